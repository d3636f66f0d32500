// philox.cuh -- Philox4x32-10 counter-based generator for the native RNG mode.
//
// The north_star's "native" random stream: a counter-based Philox generator
// keyed by (trial, node, step), next to the replay mode that regenerates the
// reference's own splitmix counter hash (streams.py:29-55).  Philox4x32-10
// (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3"):
// a 128-bit counter and a 64-bit key, ten rounds of
//   (hi0, lo0) = M0 * c0,  (hi1, lo1) = M1 * c2,
//   c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0),   k += (W0, W1) between rounds.
// Known-answer vectors: tests/test_native_abi.py (host build) and
// tests/test_gpu_parity.py (device build); the oracle restates it separately.
//
// Native-mode draw of trial k (global index), node i, sub-step counter c:
//   X = philox4x32_10(ctr = {i, c, k >> 2, tag}, key = native seed)[k & 3]
//   u = (X + 1/2) 2^-32,  r = 2u - 1 = (2X + 1) 2^-32 - 1   (exact in fp64)
// so four trials of a word share one Philox call.  The SpSA stall draw is the
// same with tag 4: stall iff (X + 1/2) 2^-32 < p_stall.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define PB_HD __host__ __device__ __forceinline__
#else
#define PB_HD inline
#endif

namespace pbsa {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;
constexpr uint32_t kNativeTagR = 3u;      // activation draw (same tag number as streams.TAG_R)
constexpr uint32_t kNativeTagStall = 4u;  // SpSA stall draw (streams.TAG_STALL)

PB_HD uint32_t philox_mulhi(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

// Philox4x32-10 of counter (c0, c1, c2, c3) under key (k0, k1).
PB_HD void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                         uint32_t k1, uint32_t (&out)[4]) {
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = philox_mulhi(kPhiloxM0, c0), lo0 = kPhiloxM0 * c0;
        const uint32_t hi1 = philox_mulhi(kPhiloxM1, c2), lo1 = kPhiloxM1 * c2;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

// Same with the ten round keys precomputed, rk[2r], rk[2r+1] = key + r (W0, W1):
// a kernel passes them in its parameter block, so each key is a constant-bank
// operand of the round's LOP3 instead of a register.
PB_HD void philox4x32_10_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                            const uint32_t (&rk)[20], uint32_t (&out)[4]) {
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = philox_mulhi(kPhiloxM0, c0), lo0 = kPhiloxM0 * c0;
        const uint32_t hi1 = philox_mulhi(kPhiloxM1, c2), lo1 = kPhiloxM1 * c2;
        c0 = hi1 ^ c1 ^ rk[2 * r];
        c1 = lo1;
        c2 = hi0 ^ c3 ^ rk[2 * r + 1];
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

PB_HD void philox_round_keys(uint32_t k0, uint32_t k1, uint32_t (&rk)[20]) {
    for (int r = 0; r < 10; ++r) {
        rk[2 * r] = k0 + (uint32_t)r * kPhiloxW0;
        rk[2 * r + 1] = k1 + (uint32_t)r * kPhiloxW1;
    }
}

// The native draw X of one trial (global index k) at node i, counter c.
PB_HD uint32_t native_draw(uint32_t k0, uint32_t k1, uint64_t k, uint32_t i, uint32_t c,
                           uint32_t tag) {
    uint32_t o[4];
    philox4x32_10(i, c, (uint32_t)(k >> 2), tag, k0, k1, o);
    return o[k & 3];
}

}  // namespace pbsa
