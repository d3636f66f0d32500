// libm_tanh.cuh -- fp64 tanh that rounds exactly like the host libm the
// reference runs on, usable on both the device (sm_100a) and the host.
//
// Why: the reference decides every p-bit update with
//     act = r + tanh(lam * (inp + delta)) >= 0        (_kernels.py:150-152)
// where tanh is the process's libm (numba lowers math.tanh to the C symbol).
// CUDA's own tanh() differs from it in the last ulp for some inputs, which
// would flip decisions whenever |r + tanh| is within an ulp of zero and so
// break bit-exact replay.  This header restates the libm algorithm
// operation-for-operation instead:
//   * tanh: the classic fdlibm reduction (tanh via expm1 of 2|x|),
//     which glibc 2.39 compiles without FMA;
//   * expm1: the x86-64 FMA/AVX2 multiarch variant that glibc selects on
//     every CPU with FMA+AVX2 (both the build container and the B200 hosts).
//     Its fused multiply-adds were read off the shipped libm.so.6 and are
//     reproduced with explicit fma(); every other operation is a single
//     IEEE-rounded add/sub/mul/div with contraction disabled.
// Parity: tests/test_native_abi.py::test_host_tanh_port_equals_libm compares
// pbsa_libm_tanh_host() (this code,
// compiled for the host) with the system tanh on millions of inputs, and the
// GPU tests (test_gpu_parity.py::test_device_tanh_matches_host_libm) compare
// the device build against the same host values.
#pragma once
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define PB_HD __host__ __device__ __forceinline__
#else
#define PB_HD static inline
#include <math.h>
#endif

#if defined(__CUDA_ARCH__)
#define PB_ADD(a, b) __dadd_rn((a), (b))
#define PB_SUB(a, b) __dsub_rn((a), (b))
#define PB_MUL(a, b) __dmul_rn((a), (b))
#define PB_DIV(a, b) __ddiv_rn((a), (b))
#define PB_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
// Host: the translation unit is compiled with -ffp-contract=off.
#define PB_ADD(a, b) ((a) + (b))
#define PB_SUB(a, b) ((a) - (b))
#define PB_MUL(a, b) ((a) * (b))
#define PB_DIV(a, b) ((a) / (b))
#define PB_FMA(a, b, c) fma((a), (b), (c))
#endif

PB_HD uint64_t pb_bits(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, sizeof u);
    return u;
#endif
}

PB_HD double pb_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, sizeof x);
    return x;
#endif
}

// Add k to the binary exponent by integer arithmetic on the high word, as
// the libm code does (no rounding involved).
PB_HD double pb_add_exponent(double y, int k) {
    uint64_t u = pb_bits(y);
    uint32_t hi = (uint32_t)(u >> 32) + ((uint32_t)k << 20);
    return pb_from_bits(((uint64_t)hi << 32) | (u & 0xffffffffULL));
}

// expm1 for finite |x| < 709.78 (the only range tanh ever passes in).
PB_HD double pb_libm_expm1(double x) {
    const double kInvLn2 = 1.4426950408889634;         // 0x3ff71547652b82fe
    const double kLn2Hi = 6.93147180369123816490e-01;  // 0x3fe62e42fee00000
    const double kLn2Lo = 1.90821492927058770002e-10;  // 0x3dea39ef35793c76
    const double kQ1 = -3.33333333333331316428e-02;
    const double kQ2 = 1.58730158725481460165e-03;
    const double kQ3 = -7.93650757867487942473e-05;
    const double kQ4 = 4.00821782732936239552e-06;
    const double kQ5 = -2.01099218183624371326e-07;

    const uint32_t top = (uint32_t)(pb_bits(x) >> 32);
    const uint32_t neg = top & 0x80000000u;
    const uint32_t hx = top & 0x7fffffffu;
    double c = 0.0;
    int k;
    if (hx > 0x40436879u && neg) return PB_SUB(1.0e-300, 1.0);  // x <= -56 ln2
    if (hx > 0x3fd62e42u) {          // |x| > ln2 / 2
        double hi, lo;
        if (hx > 0x3ff0a2b1u) {      // |x| >= 1.5 ln2: k = nearest(x / ln2)
            const double half = neg ? -0.5 : 0.5;
            k = (int)PB_ADD(half, PB_MUL(x, kInvLn2));
            const double t = (double)k;
            hi = PB_FMA(-t, kLn2Hi, x);
            lo = PB_MUL(t, kLn2Lo);
        } else if (!neg) {
            hi = PB_SUB(x, kLn2Hi); lo = kLn2Lo; k = 1;
        } else {
            hi = PB_ADD(x, kLn2Hi); lo = -kLn2Lo; k = -1;
        }
        x = PB_SUB(hi, lo);
        c = PB_SUB(PB_SUB(hi, x), lo);
    } else if (hx <= 0x3c8fffffu) {  // |x| < 2^-54: expm1(x) rounds to x
        return x;
    } else {
        k = 0;
    }

    const double hfx = PB_MUL(x, 0.5);
    const double hxs = PB_MUL(x, hfx);
    const double R2 = PB_FMA(hxs, kQ3, kQ2);
    const double R3 = PB_FMA(hxs, kQ5, kQ4);
    const double h2 = PB_MUL(hxs, hxs);
    const double R1 = PB_FMA(hxs, kQ1, 1.0);
    const double h4 = PB_MUL(h2, h2);
    const double r1 = PB_FMA(h4, R3, PB_FMA(h2, R2, R1));
    const double t = PB_FMA(-r1, hfx, 3.0);
    double e = PB_MUL(PB_DIV(PB_SUB(r1, t), PB_FMA(-x, t, 6.0)), hxs);
    if (k == 0) return PB_SUB(x, PB_FMA(e, x, -hxs));
    e = PB_SUB(PB_FMA(PB_SUB(e, c), x, -c), hxs);
    if (k == -1) return PB_FMA(0.5, PB_SUB(x, e), -0.5);
    if (k == 1) {
        if (x < -0.25) return PB_MUL(PB_SUB(e, PB_ADD(x, 0.5)), -2.0);
        return PB_FMA(PB_SUB(x, e), 2.0, 1.0);
    }
    if (k <= -2 || k > 56) {
        const double y = PB_SUB(1.0, PB_SUB(e, x));
        return PB_SUB(pb_add_exponent(y, k), 1.0);
    }
    if (k < 20) {
        const double t1 = pb_from_bits((uint64_t)(0x3ff00000u - (0x200000u >> k)) << 32);
        return pb_add_exponent(PB_SUB(t1, PB_SUB(e, x)), k);
    }
    const double t2 = pb_from_bits((uint64_t)((uint32_t)(0x3ff - k) << 20) << 32);
    return pb_add_exponent(PB_ADD(PB_SUB(x, PB_ADD(e, t2)), 1.0), k);
}

// tanh for finite x (fdlibm structure, no FMA).
PB_HD double pb_libm_tanh(double x) {
    const uint64_t bits = pb_bits(x);
    const uint32_t top = (uint32_t)(bits >> 32);
    const uint32_t ix = top & 0x7fffffffu;
    double z;
    if (ix > 0x4035ffffu) {  // |x| >= 22 (also inf; NaN never reaches here)
        if (ix > 0x7fefffffu) return x != x ? PB_ADD(x, x) : (top >> 31 ? -1.0 : 1.0);
        z = PB_SUB(1.0, 1.0e-300);
    } else {
        if ((ix | (uint32_t)bits) == 0) return x;      // +-0
        if (ix <= 0x3c7fffffu) return PB_MUL(PB_ADD(1.0, x), x);  // |x| < 2^-55
        const double ax = pb_from_bits(bits & 0x7fffffffffffffffULL);
        if (ix > 0x3fefffffu) {  // |x| >= 1
            const double t = pb_libm_expm1(PB_ADD(ax, ax));
            z = PB_SUB(1.0, PB_DIV(2.0, PB_ADD(t, 2.0)));
        } else {
            const double t = pb_libm_expm1(PB_MUL(ax, -2.0));
            z = PB_DIV(-t, PB_ADD(t, 2.0));
        }
    }
    return (top >> 31) ? -z : z;
}
