// dispatch.h -- host-side kernel selection.  The sweep kernels are templates
// on the count width L (degree < 2^L); each L is instantiated in its own
// translation unit (kernels_L<1..7>.cu, built in parallel) and plan.cu picks
// the function pointer for a plan through these declarations.
#pragma once
#include "device_common.cuh"

namespace pbsa_dispatch {

using PackedKernel = void (*)(pbsa::PackedArgs);
using ResidentKernel = void (*)(pbsa::ResidentArgs);
using ResidentTimingKernel = void (*)(pbsa::ResidentTimingArgs);

// var: 0 ideal profile, 1 varied profile without timing spread, 2 with one
template <int L>
PackedKernel packed_kernel(bool update, bool cached, bool tapsa, bool spsa, int var, bool native);
template <int L>
ResidentKernel resident_kernel(bool cached, bool varu, bool native, bool tapsa);
template <int L>
ResidentTimingKernel resident_timing_kernel(bool native);
// the timing-spread sweep over period buckets (packed_sweep_bucket)
template <int L>
PackedKernel bucket_kernel(bool native);

}  // namespace pbsa_dispatch
