// kernels_L.cuh -- definitions of the dispatch.h selectors; included by the
// per-L translation units kernels_L<1..7>.cu, which instantiate one L each.
#pragma once
#include "dispatch.h"
#include "packed_kernels.cuh"
#include "resident_kernels.cuh"

namespace pbsa_dispatch {

template <int L>
PackedKernel packed_kernel(bool update, bool cached, bool tapsa, bool spsa, int var, bool native) {
    if (!update) return pbsa::packed_sweep<L, false, false>;
    if (native) {  // Philox draws (no first-absorb cache)
        if (var) return var == 2 ? pbsa::packed_sweep_timing<L, true> : pbsa::packed_sweep<L, true, false, 5>;
        if (tapsa) return pbsa::packed_sweep<L, true, false, 6>;
        if (spsa) return pbsa::packed_sweep<L, true, false, 7>;
        return pbsa::packed_sweep<L, true, false, 4>;
    }
    if (var)
        return var == 2 ? pbsa::packed_sweep_timing<L>
                        : cached ? pbsa::packed_sweep<L, true, true, 3> : pbsa::packed_sweep<L, true, false, 3>;
    if (tapsa) return cached ? pbsa::packed_sweep<L, true, true, 1> : pbsa::packed_sweep<L, true, false, 1>;
    if (spsa) return cached ? pbsa::packed_sweep<L, true, true, 2> : pbsa::packed_sweep<L, true, false, 2>;
    return cached ? pbsa::packed_sweep<L, true, true> : pbsa::packed_sweep<L, true, false>;
}

template <int L>
ResidentKernel resident_kernel(bool cached, bool varu, bool native, bool tapsa) {
    if (tapsa)
        return native ? pbsa::resident_sweep<L, false, false, true, true>
                      : (cached ? pbsa::resident_sweep<L, true, false, false, true>
                                : pbsa::resident_sweep<L, false, false, false, true>);
    if (native) return varu ? pbsa::resident_sweep<L, false, true, true> : pbsa::resident_sweep<L, false, false, true>;
    if (varu) return cached ? pbsa::resident_sweep<L, true, true> : pbsa::resident_sweep<L, false, true>;
    return cached ? pbsa::resident_sweep<L, true, false> : pbsa::resident_sweep<L, false, false>;
}

template <int L>
ResidentTimingKernel resident_timing_kernel(bool native) {
    return native ? pbsa::resident_timing<L, true> : pbsa::resident_timing<L, false>;
}

template <int L>
PackedKernel bucket_kernel(bool native) {
    return native ? pbsa::packed_sweep_bucket<L, true> : pbsa::packed_sweep_bucket<L, false>;
}

}  // namespace pbsa_dispatch

#define PBSA_INSTANTIATE_L(l)                                                                            \
    template pbsa_dispatch::PackedKernel pbsa_dispatch::packed_kernel<l>(bool, bool, bool, bool, int, bool); \
    template pbsa_dispatch::ResidentKernel pbsa_dispatch::resident_kernel<l>(bool, bool, bool, bool);      \
    template pbsa_dispatch::ResidentTimingKernel pbsa_dispatch::resident_timing_kernel<l>(bool);           \
    template pbsa_dispatch::PackedKernel pbsa_dispatch::bucket_kernel<l>(bool);
