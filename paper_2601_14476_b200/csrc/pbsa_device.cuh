// pbsa_device.cuh -- device kernels of the B200-native pSA sweep.
//
// Restates, for sm_100a, the reference hot loop
//   /root/reference/pkg/src/pbitsa/_kernels.py:68-175  (anneal_loop)
// batched over trials.  Two paths:
//
//  * PACKED (the production path for MAX-CUT-shaped work: J in {+1,-1}, h = 0,
//    ideal profile, plain pSA rule).  Spins are bit-packed, 32 trials per
//    uint32 word, layout [node][word]; one thread owns one (node, word) task
//    = 32 p-bit updates.  The local field of all 32 trials is formed with a
//    bit-sliced adder over the neighbour words; the activation is an exact
//    integer threshold on the 64-bit counter hash (thresholds derived on the
//    host from libm-exact tanh per (cycle, raw field)), so no tanh runs on the
//    device and the result is bit-identical to the reference.  The per-cycle
//    cut is fused into the next sweep's gather (sum_i s_i raw_i).
//
//  * GENERAL (any real J/h, any variability profile, all three input rules).
//    int8 spins, layout [node][trial]; one thread per (node, trial); fp64
//    arithmetic in the reference's exact operation order with contraction
//    disabled, and a tanh that rounds like the host libm (libm_tanh.cuh).
//
// Both paths draw every random number from the same splitmix-style counter
// hash as streams.py:29-55, regenerated in-kernel from (key, tag, node, count).
#pragma once
#include <cooperative_groups.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "libm_tanh.cuh"
#include "philox.cuh"

#define PB_GAMMA 0x9E3779B97F4A7C15ULL
#define PB_M1 0xBF58476D1CE4E5B9ULL
#define PB_M2 0x94D4A04C32684F87ULL

namespace pbsa {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * PB_M1;
    z = (z ^ (z >> 27)) * PB_M2;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t absorb(uint64_t h, uint64_t w) {
    return mix64((h + PB_GAMMA) ^ w);
}

// u01 = (h >> 11) * 2^-53 exactly (streams.py:48-50).
__device__ __forceinline__ double u01_of(uint64_t h) {
    return __dmul_rn(__ull2double_rn(h >> 11), 0x1p-53);
}

// ------------------------------------------------------------------ init
// Initial spins: u01(key, TAG_SPIN, i, 0) < 0.5  <=>  stream word < 2^63
// (_kernels.py:94-97).  kspin[t] = absorb(key_t, TAG_SPIN) (host prefix).

__global__ void init_packed(uint32_t *__restrict__ s, const uint64_t *__restrict__ kspin,
                            int n, int W) {
    const int64_t task = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (task >= (int64_t)n * W) return;
    const int w = (int)(task / n), i = (int)(task % n);
    uint32_t word = 0;
#pragma unroll 4
    for (int b = 0; b < 32; ++b) {
        const uint64_t h = absorb(absorb(kspin[w * 32 + b], (uint64_t)i), 0);
        word |= (uint32_t)((h >> 63) == 0) << b;
    }
    s[task] = word;
}

__global__ void init_general(int8_t *__restrict__ s, const uint64_t *__restrict__ kspin, int n,
                             int Tp) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)n * Tp) return;
    const int i = (int)(g / Tp), t = (int)(g % Tp);
    const uint64_t h = absorb(absorb(kspin[t], (uint64_t)i), 0);
    s[g] = (h >> 63) == 0 ? 1 : -1;
}

// Per-(trial, node) first absorb of the TAG_R draw, which does not depend on
// the sub-step: s = absorb(K_t, i) + GAMMA (K_t = absorb(key, TAG_R)), plus the
// count-independent part of the next xorshift, stored in
// 8 KB tiles per (word w, 32-node chunk) laid out [trial b][lane] so the sweep
// reads trial b of its node at a fixed offset and every load is 256 B coalesced.
__global__ void packed_cache_init(uint2 *__restrict__ acache, const uint64_t *__restrict__ krg,
                                  int n, int chunks, int W) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)W * chunks * 1024) return;
    const int lane = (int)(g & 31), b = (int)((g >> 5) & 31);
    const int64_t tile = g >> 10;
    const int ch = (int)(tile % chunks), w = (int)(tile / chunks);
    const int i = ch * 32 + lane;
    uint64_t s = 0;
    if (i < n) s = mix64(krg[w * 32 + b] ^ (uint64_t)i) + PB_GAMMA;
    // store y' = s ^ (s >> 30): the sweep only XORs the sub-step counter into
    // its low word (count < 2^30 never reaches the shifted bits)
    const uint64_t y = s ^ (s >> 30);
    acache[g] = make_uint2((uint32_t)y, (uint32_t)(y >> 32));
}

// ---------------------------------------------------------- packed sweep
// Layout: spins uint32 [W][n] (word-major, node-fast): bit b of word (w, i) is
// trial 32w+b's spin at node i, 1 = +1.  A warp owns one word index w for its
// whole life and walks 32-node chunks of it (lane = node), so the 32 trial
// constants of the warp are uniform (broadcast from shared memory), neighbour
// words of consecutive nodes are coalesced on lattice-like graphs, and the
// per-trial cut partials reduce with one 32x32 butterfly per warp.
//
// The per-update draw is H = absorb(absorb(K, i), count) with
// K = absorb(key, TAG_R) (streams.py:41-45, _kernels.py:149).  Two exact
// algebraic reductions shorten it (both need i < 2^30 and count < 2^30, which
// the host checks before choosing this path):
//   * the first xorshift of absorb(K, i) only sees i in bits < 30, so
//     y = (F_t ^ i, Y_t) with per-trial constants, and the high word of
//     y * M1 is umulhi(y_lo, M1lo) + y_lo * M1hi + C_t with C_t = Y_t * M1lo;
//   * likewise count enters the first xorshift of the second absorb as a
//     plain XOR on the low word.
// The activation decision "H >= thr" is taken on the high word of the last
// multiply (before the final xorshift) through the carry of zhi + ~thi; the
// only inputs where that can differ from the exact 64-bit test are
// (zhi >> 1) == (thi >> 1), which flag the word for an exact recomputation.
struct PackedArgs {
    const uint32_t *sold;
    uint32_t *snew;
    const uint32_t *rowptr;   // [n+1]
    const uint32_t *adj;      // [nnz] column | (J < 0) << 31
    const uint2 *kfc;         // [Tp] per-trial (F_t, C_t)
    const uint2 *acache;      // [W][chunks][32 trials][32 lanes] absorb(K_t, i) + GAMMA, or null
    const uint64_t *krg;      // [Tp] absorb(key, TAG_R) + GAMMA (exact slow path)
    const uint64_t *thr;      // [K] thresholds of this cycle (H >= thr -> +1)
    unsigned long long *pacc; // [Tp] += sum_i s_i * raw_i of the sub-step's input state
    int16_t *raw_out;         // [n][Tp] raw field of this update, or null
    int n, W, Tp, K, dmax;
    int warps_per_word;       // warps sharing one word index
    int chunks;               // ceil(n / 32)
    uint32_t count;           // global sub-step counter c * t_res (< 2^30)
    int do_update;            // 0: only accumulate pacc (final cut pass)
    uint32_t *sidx;           // SpSA: [W][32][n] threshold-table index of each p-bit's drive
    const uint32_t *thr_hi_all;  // SpSA: [cycles][K] high words of all thresholds
    const uint2 *kfs;         // SpSA: [Tp] per-trial (F, C) of absorb(key, TAG_STALL)
    const uint64_t *kst;      // SpSA: [Tp] absorb(key, TAG_STALL) + GAMMA (exact slow path)
    const uint64_t *thr_all;  // SpSA: [cycles][K] all thresholds
    uint64_t p_stall64;       // SpSA: stall iff H_stall < p_stall64 (~0: always)
    int cycle, Kc;            // SpSA: this cycle, entries per cycle
    int sidx_full;            // SpSA: store every drive index (full sectors), not only fresh ones
    uint32_t *ring;           // TApSA: [W][alpha][L][n] bit-sliced neighbour counts
    int alpha, slot, filled;  // TApSA: ring length, this cycle's slot, min(c+1, alpha)
    // VAR (per-p-bit variability profile, plain rule)
    const float2 *prof;       // [W][32][n] {fl32(lam), fl32(lam * delta)} (no timing spread)
    const __half2 *prof16;    // [W][n][32] {fl16(lam), fl16(lam * delta)} (timing spread)
    const double *lam64;      // [W*32][n] exact lam (near-tie path)
    const double *del64;      // [W*32][n] exact delta
    const uint32_t *pplanes;  // [W][nplanes][n] bit-sliced clamped periods, or null (all fire)
    const uint8_t *divs;      // [ndiv] the present periods that divide this sub-step's counter
    int ndiv, nplanes;
    int do_cut;               // accumulate pacc (first sub-step of a cycle; always 1 off VAR)
    float i0f;                // fl32(i0) of this cycle
    float margin;             // prefilter margin scale (1; huge = every update takes the exact path)
    double i0;                // i0 of this cycle
    double *inp_out;          // [W*32][n] i0 * raw of every fired p-bit, or null
    // NATIVE (ALG=4: Philox4x32-10 draws instead of the replayed hash, philox.cuh)
    uint32_t nk0, nk1;        // Philox key (native seed)
    uint32_t rk[20];          // its ten round keys (philox_round_keys)
    uint32_t ngroup;          // Philox trial-group counter of this launch's word 0: (first trial) / 4
    int reg4;                 // every degree is 4 (rowptr[i] = 4i): gather_counts_reg4
};

// Exact H >= thr for H = mix64(x); thr == ~0 encodes "never" (tanh == -1),
// which no genuine threshold equals (their low 11 bits are clear).
__device__ __forceinline__ bool hash_ge_exact(uint64_t x, uint64_t thr) {
    return mix64(x) >= thr && thr != ~0ULL;
}

constexpr int kPackedThreads = 256;
constexpr int kPackedWarps = kPackedThreads / 32;

__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }

// First absorb of a trial's draw: s = absorb(K, i) + GAMMA, as (lo, hi).
// y = (ylo, Y) with ylo = F_t ^ i; Y * M1L is folded into C = C_t.
// Right shifts of high words go through IMAD.HI (x >> s == umulhi(x, 2^(32-s)))
// so the FMA pipe takes part of the load of the saturated ALU pipe.
__device__ __forceinline__ void packed_first_absorb(uint32_t ylo, uint32_t C, uint32_t &sl,
                                                    uint32_t &sh) {
    constexpr uint32_t M1L = 0x1CE4E5B9u, M1H = 0xBF58476Du;
    constexpr uint32_t M2L = 0x32684F87u, M2H = 0x94D4A04Cu;
    constexpr uint32_t GL = 0x7F4A7C15u, GH = 0x9E3779B9u;
    uint32_t zl = ylo * M1L;
    uint32_t zh = mulhi(ylo, M1L) + ylo * M1H + C;
    // z ^= z >> 27 ; z *= M2
    uint32_t yl = zl ^ __funnelshift_r(zl, zh, 27);
    uint32_t yh = zh ^ mulhi(zh, 1u << 5);
    zl = yl * M2L;
    zh = mulhi(yl, M2L) + yl * M2H + yh * M2L;
    // z ^= z >> 31  -> A ; s = A + GAMMA
    yl = zl ^ __funnelshift_r(zl, zh, 31);
    yh = zh ^ mulhi(zh, 1u << 1);
    asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
        : "=r"(sl), "=r"(sh) : "r"(yl), "r"(yh), "r"(GL), "r"(GH));
}

// Second absorb from y = x ^ (x >> 30), x = s ^ count, up to the high word of
// the last multiply, then the decision bit shifted into `word` through the
// carry of zh + ~thi.  Returns the (zh ^ thi) tie witness (< 2: recompute).
__device__ __forceinline__ uint32_t packed_decide_y(uint32_t yl, uint32_t yh, uint2 t,
                                                    uint32_t &word) {
    constexpr uint32_t M1L = 0x1CE4E5B9u, M1H = 0xBF58476Du;
    constexpr uint32_t M2L = 0x32684F87u, M2H = 0x94D4A04Cu;
    uint32_t zl = yl * M1L;
    uint32_t zh = mulhi(yl, M1L) + yl * M1H + yh * M1L;
    yl = zl ^ __funnelshift_r(zl, zh, 27);
    yh = zh ^ mulhi(zh, 1u << 5);
    zh = mulhi(yl, M2L) + yl * M2H + yh * M2L;
    uint32_t dummy;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %4;"
        : "=r"(dummy), "=r"(word) : "r"(zh), "r"(t.x), "r"(word));
    return zh ^ t.y;
}

// High word zh of the last multiply of the second absorb, from its input
// y = x ^ (x >> 30); the draw's top word is zh ^ (zh >> 31), within 1 of zh.
__device__ __forceinline__ uint32_t packed_hash_hi_y(uint32_t yl, uint32_t yh) {
    constexpr uint32_t M1L = 0x1CE4E5B9u, M1H = 0xBF58476Du;
    constexpr uint32_t M2L = 0x32684F87u, M2H = 0x94D4A04Cu;
    const uint32_t zl = yl * M1L;
    const uint32_t zh = mulhi(yl, M1L) + yl * M1H + yh * M1L;
    yl = zl ^ __funnelshift_r(zl, zh, 27);
    yh = zh ^ mulhi(zh, 1u << 5);
    return mulhi(yl, M2L) + yl * M2H + yh * M2L;
}

// Same from the first absorb s (x = s ^ count; count < 2^30 only touches the low word).
__device__ __forceinline__ uint32_t packed_hash_hi(uint32_t sl, uint32_t sh, uint32_t count) {
    return packed_hash_hi_y(sl ^ count ^ __funnelshift_r(sl, sh, 30), sh ^ mulhi(sh, 1u << 2));
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Variability prefilter on the fp16 profile pair (fl16(lam), fl16(lam delta)).
// The computed x = fl16(lam) ir + fl16(lam delta) is within
//   dx <= A 2^-10.9 + 2^-22,   A = |lam| |i0 raw| + |lam delta|,
// of the reference's fp64 x (fp16 rounding 2^-11 each, ir and fma in fp32).  On
// [x - dx, x + dx] the slope of t*(x) = 1/(1 + e^{2x}) is at most
// 2 q e^{2 dx}, q = t(1 - t) at x (cosh(x + dx) >= cosh(x) e^{-dx}), so with
// A <= 256 (e^{2 dx} <= 1.35) the threshold moves by at most
// q (5.93e6 A + 2765) units of 2^-32; the fp32 evaluation of t and of
// zh - t 2^32 adds at most (A + 1) 2^11 + 2^9 (the fp32-profile analysis).
// Hence |zh - t 2^32| >= M = A 2^11 + 5120 + 6.3e6 q A decides exactly;
// otherwise (and for A > 256, or a non-finite pair) the update takes the exact
// fp64 recheck.  Returns diff > 0 in bit 0 and "undecided" in bit 1.
// The same on the fp32 pair (fl32(lam), fl32(lam delta)) -- the kernels without
// a timing spread, whose profile reads are coalesced: |x - x64| <= A 2^-21.9,
// so M = (A + 2) 2^11 (module comment of packed_sweep) and only ~2^-16 of the
// updates take the recheck.
__device__ __forceinline__ uint32_t var_prefilter(float2 lv, float ir, uint32_t zh, float ms) {
    const float x = fmaf(lv.x, ir, lv.y);
    const float A = fmaf(fabsf(lv.x), fabsf(ir), fabsf(lv.y));
    const float t = rcp_approx(1.0f + ex2_approx(x * 2.88539008f));
    const float diff = fmaf(-t, 4294967296.0f, __uint2float_rn(zh));
    const bool undecided = !(fabsf(diff) >= ms * fmaf(A, 2048.0f, 4096.0f));
    return (undecided ? 2u : 0u) | (diff > 0.0f ? 1u : 0u);
}

__device__ __forceinline__ uint32_t var_prefilter(__half2 h, float ir, uint32_t zh, float ms) {
    const float2 lv = __half22float2(h);
    const float x = fmaf(lv.x, ir, lv.y);
    const float A = fmaf(fabsf(lv.x), fabsf(ir), fabsf(lv.y));
    const float t = rcp_approx(1.0f + ex2_approx(x * 2.88539008f));
    const float q = fmaf(-t, t, t);
    const float M = ms * fmaf(6.3e6f * q, A, fmaf(A, 2048.0f, 5120.0f));
    const float diff = fmaf(-t, 4294967296.0f, __uint2float_rn(zh));
    const bool undecided = !(fabsf(diff) >= M) || !(A <= 256.0f);
    return (undecided ? 2u : 0u) | (diff > 0.0f ? 1u : 0u);
}

// Second absorb (x = s ^ count; count < 2^30 only touches the low word).
__device__ __forceinline__ uint32_t packed_second_decide(uint32_t sl, uint32_t sh, uint32_t count,
                                                         uint2 t, uint32_t &word) {
    return packed_decide_y(sl ^ count ^ __funnelshift_r(sl, sh, 30), sh ^ mulhi(sh, 1u << 2), t,
                           word);
}

// Plain-rule variant with the table entry t = (lo, hi) of the 33-bit
// n2 = ~thi + 2: the carry of zh + n2 is zh >= thi - 1 and its low word is
// D = zh - thi + 1, so D < 3 (zh within 1 of thi, where the draw's low word
// or the final xorshift's bit 0 matter) is the only case that needs the
// exact 64-bit test, and every other carry is the exact decision -- also for
// thi <= 1, which the 33rd bit keeps.  Returns D.
__device__ __forceinline__ uint32_t packed_decide_n2(uint32_t yl, uint32_t yh, uint2 t,
                                                     uint32_t &word) {
    constexpr uint32_t M1L = 0x1CE4E5B9u, M1H = 0xBF58476Du;
    constexpr uint32_t M2L = 0x32684F87u, M2H = 0x94D4A04Cu;
    uint32_t zl = yl * M1L;
    uint32_t zh = mulhi(yl, M1L) + yl * M1H + yh * M1L;
    yl = zl ^ __funnelshift_r(zl, zh, 27);
    yh = zh ^ mulhi(zh, 1u << 5);
    zh = mulhi(yl, M2L) + yl * M2H + yh * M2L;
    uint32_t D;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
        : "=r"(D), "=r"(word) : "r"(zh), "r"(t.x), "r"(word), "r"(word + t.y));
    return D;
}

__device__ __forceinline__ uint32_t packed_second_decide_n2(uint32_t sl, uint32_t sh, uint32_t count,
                                                            uint2 t, uint32_t &word) {
    return packed_decide_n2(sl ^ count ^ __funnelshift_r(sl, sh, 30), sh ^ mulhi(sh, 1u << 2), t,
                            word);
}

// Native decision: shift (X >= T) into `word` as the carry of X + (2^32 - T),
// t = (lo, hi) of the 33-bit 2^32 - T (T = 2^32 never fires, T = 0 always).
__device__ __forceinline__ void native_decide(uint32_t X, uint2 t, uint32_t &word) {
    uint32_t dummy;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
        : "=r"(dummy), "=r"(word) : "r"(X), "r"(t.x), "r"(word), "r"(word + t.y));
}

// Bit-sliced counter: add the L-bit per-trial numbers x[] into C[] (CL planes).
template <int L, int CL>
__device__ __forceinline__ void vc_add(uint32_t (&C)[CL], const uint32_t (&x)[L]) {
    uint32_t carry = 0;
#pragma unroll
    for (int r = 0; r < CL; ++r) {
        const uint32_t v = r < L ? x[r] : 0u;
        const uint32_t s = C[r] ^ v ^ carry;
        carry = (C[r] & v) | (carry & (C[r] ^ v));
        C[r] = s;
    }
}

// Per-thread cut counter width for degree < 2^L: L + 2 planes, so one lane
// may take up to 4 nodes (the host sizes warps per word accordingly).
template <int L>
struct CutPlanes {
    static constexpr int value = L + 2;
};

#ifndef PBSA_PACKED_MIN_BLOCKS
#define PBSA_PACKED_MIN_BLOCKS 4
#endif

// TApSA (time-averaged rule, _kernels.py:131-138) on the packed path: every
// p-bit fires once per cycle, so the history slot (c % alpha) and the fill
// count min(c+1, alpha) are the same for the whole launch.  The ring keeps the
// bit-sliced neighbour counts p of the last alpha cycles ([W][alpha][L][n]);
// the drive is i0 * (acc / filled) with acc = 2 S - filled * d and
// S = sum of p over the filled slots (< 64), so the threshold is a per-cycle
// table lookup by (degree, S), exactly like the plain rule.

// Bit-sliced count p = #{J_ik s_k = +1} (the local field, raw = 2p - d) of
// the 32 trials over the neighbours [beg, end) of one node.
// Carry-save adder: (h, l) = a + b + l as bit-sliced digits (two LOP3s).
__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b) {
    const uint32_t u = l ^ a;
    h = (l & a) | (u & b);
    l = u ^ b;
}

// Bit-sliced count over neighbours [beg, end), the neighbour word of entry k
// given by nb(k).  Degrees >= 8 go through a Harley-Seal carry-save tree
// (seven CSAs per eight neighbours, ~2 ops each, plus one ripple of the
// weight-8 digit) instead of an L-plane ripple per neighbour.
template <int L, typename NB>
__device__ __forceinline__ void count_neighbours(uint32_t beg, uint32_t end, NB nb, uint32_t (&p)[L]) {
#pragma unroll
    for (int r = 0; r < L; ++r) p[r] = 0;
    auto ripple = [&](uint32_t cp, int from) {
#pragma unroll
        for (int r = 0; r < L; ++r) {
            if (r < from) continue;
            const uint32_t np = p[r] & cp;
            p[r] ^= cp;
            cp = np;
        }
    };
    uint32_t k = beg;
    if (L >= 4) {
        for (; k + 8 <= end; k += 8) {
            uint32_t x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = nb(k + j);
            uint32_t twosA, twosB, foursA, foursB, eights;
            csa(twosA, p[0], x[0], x[1]);
            csa(twosB, p[0], x[2], x[3]);
            csa(foursA, p[1], twosA, twosB);
            csa(twosA, p[0], x[4], x[5]);
            csa(twosB, p[0], x[6], x[7]);
            csa(foursB, p[1], twosA, twosB);
            csa(eights, p[2], foursA, foursB);
            ripple(eights, 3);
        }
    }
    for (; k < end; ++k) ripple(nb(k), 0);
}

template <int L>
__device__ __forceinline__ void gather_counts(const uint32_t *__restrict__ adj,
                                              const uint32_t *__restrict__ sw, uint32_t beg,
                                              uint32_t end, uint32_t (&p)[L]) {
    count_neighbours<L>(beg, end, [&](uint32_t k) {
        const uint32_t e = __ldg(adj + k);
        return __ldg(sw + (e & 0x7fffffffu)) ^ (uint32_t)((int32_t)e >> 31);
    }, p);
}

// Degree-4 regular graphs (the G-set tori): node i's entries sit at 4i, so the
// row needs no rowptr load and its four entries come in one 16-byte load --
// one dependent global load fewer in front of the neighbour gather.
template <int L>
__device__ __forceinline__ void gather_counts_row4(const uint4 e, const uint32_t *__restrict__ sw,
                                                   uint32_t (&p)[L]) {
    const uint32_t x0 = __ldg(sw + (e.x & 0x7fffffffu)) ^ (uint32_t)((int32_t)e.x >> 31);
    const uint32_t x1 = __ldg(sw + (e.y & 0x7fffffffu)) ^ (uint32_t)((int32_t)e.y >> 31);
    const uint32_t x2 = __ldg(sw + (e.z & 0x7fffffffu)) ^ (uint32_t)((int32_t)e.z >> 31);
    const uint32_t x3 = __ldg(sw + (e.w & 0x7fffffffu)) ^ (uint32_t)((int32_t)e.w >> 31);
    // bit-sliced x0 + x1 + x2 + x3 (<= 4 < 2^L, L >= 3 since dmax = 4)
    const uint32_t s01 = x0 ^ x1, c01 = x0 & x1, s23 = x2 ^ x3, c23 = x2 & x3;
    const uint32_t s = s01 ^ s23, cs = s01 & s23;     // weight-1 digit and its carry
    const uint32_t t = c01 ^ c23 ^ cs;                 // weight-2 digit
    const uint32_t f = (c01 & c23) | (cs & (c01 ^ c23));  // weight-4 digit
#pragma unroll
    for (int r = 0; r < L; ++r) p[r] = r == 0 ? s : r == 1 ? t : r == 2 ? f : 0u;
}

template <int L>
__device__ __forceinline__ void gather_counts_reg4(const uint32_t *__restrict__ adj,
                                                   const uint32_t *__restrict__ sw, int i,
                                                   uint32_t (&p)[L]) {
    gather_counts_row4<L>(__ldg(reinterpret_cast<const uint4 *>(adj) + i), sw, p);
}

// Cut count g = #{J_ik s_i s_k = +1} = (s_i = +1) ? p : d - p, bit-sliced:
// d - p = ~p + (d + 1) mod 2^L (p <= d < 2^L), then a per-trial select.
template <int L>
__device__ __forceinline__ void cut_counts(const uint32_t (&p)[L], uint32_t own, int d,
                                           uint32_t (&g)[L]) {
    const uint32_t dp1 = (uint32_t)(d + 1);
    uint32_t carry = 0;
#pragma unroll
    for (int r = 0; r < L; ++r) {
        const uint32_t m = 0u - ((dp1 >> r) & 1u);
        const uint32_t x = ~p[r];
        const uint32_t sum = x ^ m ^ carry;
        carry = (x & m) | (carry & (x ^ m));
        g[r] = (p[r] & own) | (sum & ~own);
    }
}

// Warp-level bit-sliced add of the 32 lanes' cut counters (all lanes of the
// warp hold the same 32 trials), then lane b adds trial 32w+b's partial.
// After butterfly round j the sums of 2^(j+1) lanes need CP + j + 1 planes,
// so each round adds only the planes that can be non-zero.
template <int CP>
__device__ __forceinline__ void warp_cut_flush(const uint32_t (&C)[CP], int dsum, int lane,
                                               unsigned long long *pacc_w) {
    uint32_t W[CP + 5];
#pragma unroll
    for (int r = 0; r < CP + 5; ++r) W[r] = r < CP ? C[r] : 0u;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int off = 16 >> j;
        uint32_t carry = 0;
#pragma unroll
        for (int r = 0; r < CP + j + 1; ++r) {
            const uint32_t o = r < CP + j ? __shfl_xor_sync(0xffffffffu, W[r], off) : 0u;
            const uint32_t sum = W[r] ^ o ^ carry;
            carry = (W[r] & o) | (carry & (W[r] ^ o));
            W[r] = sum;
        }
        dsum += __shfl_xor_sync(0xffffffffu, dsum, off);
    }
    int acc0 = 0;
#pragma unroll
    for (int r = 0; r < CP + 5; ++r) acc0 |= (int)((W[r] >> lane) & 1u) << r;
    const int acc = 2 * acc0 - dsum;
    if (pacc_w && acc) atomicAdd(pacc_w + lane, (unsigned long long)(long long)acc);
}

// Variability near-ties: the reference's fp64 arithmetic (_kernels.py:150-152)
// on the full 64-bit draw, for the trials flagged in `exact`.
// NATIVE: the same on the Philox draw, r = (2X + 1) 2^-32 - 1 (philox.cuh).
template <int L, bool NATIVE = false>
__device__ __forceinline__ uint32_t var_exact_bits(const PackedArgs &a, uint32_t exact, const uint32_t (&p)[L],
                                                int d, int w, int i, uint32_t count) {
    uint32_t word = 0;
    while (exact) {
        const int b = __ffs(exact) - 1;
        exact &= exact - 1;
        int pop = 0;
        for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
        const size_t idx = ((size_t)w * 32 + b) * a.n + i;
        double r;
        if (NATIVE) {
            uint32_t o[4];
            philox4x32_10_rk((uint32_t)i, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                             kNativeTagR, a.rk, o);
            const uint32_t x = (b & 2) ? ((b & 1) ? o[3] : o[2]) : ((b & 1) ? o[1] : o[0]);
            r = __dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(2.0, (double)x), 1.0), 0x1p-32), 1.0);
        } else {
            const uint64_t x1 = (a.krg[(size_t)w * 32 + b]) ^ (uint64_t)(uint32_t)i;
            const uint64_t x2 = (mix64(x1) + PB_GAMMA) ^ (uint64_t)count;
            r = __dsub_rn(__dmul_rn(2.0, u01_of(mix64(x2))), 1.0);
        }
        const double inp = __dmul_rn(a.i0, (double)(2 * pop - d));
        const double xx = __dmul_rn(a.lam64[idx], __dadd_rn(inp, a.del64[idx]));
        word |= (uint32_t)(__dadd_rn(r, pb_libm_tanh(xx)) >= 0.0) << b;
    }
    return word;
}

template <int L, bool UPDATE, bool CACHED, int ALG = 0>
__global__ void __launch_bounds__(kPackedThreads, PBSA_PACKED_MIN_BLOCKS) packed_sweep(PackedArgs a) {
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ unsigned long long smem_u64[];
    // Threshold table, 128 B aligned.  L <= 4 (degree <= 15): one 16-entry row
    // per degree d indexed by the neighbour count p (raw = 2p - d), so a
    // trial's entry address is (p * 8) | row base, formed with one LOP3.
    // Larger degrees: entries indexed by raw + dmax.  TApSA: 64-entry rows by S.
    // ALG: 0 plain, 1 TApSA, 2 SpSA, 3 varied profile (replayed hash);
    // 4 plain, 5 varied, 6 TApSA, 7 SpSA with Philox draws (philox.cuh)
    constexpr bool TAPSA = ALG == 1 || ALG == 6;
    constexpr bool SPSA = ALG == 2 || ALG == 7;
    constexpr bool VAR = ALG == 3 || ALG == 5;
    constexpr bool NATIVE = ALG >= 4;
    constexpr bool NIB = L <= 4 && !TAPSA;
    uint2 *sthr = reinterpret_cast<uint2 *>(
        (reinterpret_cast<uintptr_t>(smem_u64) + 511) & ~(uintptr_t)511);
    const int tab_entries = VAR ? 0 : TAPSA ? a.K : NIB ? (a.dmax + 1) * 16 : a.K;
    uint2 *skey = sthr + tab_entries;                     // [warps][32] {F, C}

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gwarp = blockIdx.x * kPackedWarps + wib;
    const int w = gwarp / a.warps_per_word;
    const int q = gwarp % a.warps_per_word;
    const bool live = w < a.W;

    for (int k = threadIdx.x; k < tab_entries; k += blockDim.x) {
        uint32_t thi;
        uint64_t tfull = 0;  // NATIVE: the 33-bit Philox threshold T
        if (TAPSA) {
            tfull = a.thr[k];  // host table is already [acc + f dmax]
            thi = (uint32_t)(tfull >> 32);
        } else {
            int raw = k - a.dmax;
            bool ok = true;
            if (NIB) {
                const int d = k >> 4, pp = k & 15;
                raw = 2 * pp - d;
                ok = pp <= d;
            }
            tfull = ok ? a.thr[raw + a.dmax] : 0ULL;
            thi = (uint32_t)(tfull >> 32);
        }
        if (NATIVE && !VAR) {  // (lo, hi) of the 33-bit 2^32 - T: carry of X + it is X >= T
            const uint64_t nt = (1ULL << 32) - tfull;
            sthr[k] = make_uint2((uint32_t)nt, (uint32_t)(nt >> 32));
        } else if (ALG == 0) {  // (lo, hi) of the 33-bit ~thi + 2 (packed_decide_n2)
            const uint64_t n2 = (uint64_t)(~thi) + 2u;
            sthr[k] = make_uint2((uint32_t)n2, (uint32_t)(n2 >> 32));
        } else {
            sthr[k] = make_uint2(~thi, thi);
        }
    }
    uint2 *key = skey + wib * 32;
    key[lane] = live ? a.kfc[(size_t)w * 32 + lane] : make_uint2(0, 0);
    // SpSA: the per-trial constants of the stall stream, likewise per warp
    uint2 *skeys = skey + kPackedWarps * 32;
    if (SPSA) skeys[wib * 32 + lane] = live ? a.kfs[(size_t)w * 32 + lane] : make_uint2(0, 0);
    uint32_t *scount = reinterpret_cast<uint32_t *>(skeys + kPackedWarps * 32);
    if (threadIdx.x == 0) scount[0] = a.count;
    __syncthreads();
    // Programmatic dependent launch: everything above reads only host-written
    // constants, so it overlaps the previous sub-step's tail; the spin state
    // of that sub-step is read only after its grid has completed.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // read back through shared memory so the counter lives in a vector
    // register (a kernel-parameter operand is re-fetched with LDCU per trial)
    const uint32_t count = scount[0];

    // Per-trial sum over this thread's nodes of q_i = #{k : J_ik s_i s_k = +1},
    // kept bit-sliced; s_i raw_i = 2 q_i - d_i, so the cut partial is
    // 2 * C - dsum (h = 0).
    constexpr int CP = CutPlanes<L>::value;
    uint32_t C[CP];
#pragma unroll
    for (int r = 0; r < CP; ++r) C[r] = 0;
    int dsum = 0;

    if (live) {
        const uint32_t *sw = a.sold + (size_t)w * a.n;
        // degree-4 rows: the next chunk's row (one 16-byte load) and own word are
        // fetched one iteration ahead, so only the neighbour loads precede the counts
        // (only the last chunk has lanes past n, and it has no successor)
        const bool R4 = L >= 3 && a.reg4;
        const uint4 *adj4 = reinterpret_cast<const uint4 *>(a.adj);
        uint4 e_nx = make_uint4(0u, 0u, 0u, 0u);
        uint32_t own_nx = 0;
        if (R4 && q < a.chunks && q * 32 + lane < a.n) {
            e_nx = __ldg(adj4 + q * 32 + lane);
            own_nx = __ldg(sw + q * 32 + lane);
        }
        for (int ch = q; ch < a.chunks; ch += a.warps_per_word) {
            const int i = ch * 32 + lane;
            if (i >= a.n) continue;
            uint32_t p[L];
            int d;
            uint32_t own;
            if (R4) {
                const uint4 e = e_nx;
                own = own_nx;
                const int ni = i + 32 * a.warps_per_word;
                if (ni < a.n) {
                    e_nx = __ldg(adj4 + ni);
                    own_nx = __ldg(sw + ni);
                }
                gather_counts_row4<L>(e, sw, p);
                d = 4;
            } else {
                const uint32_t beg = __ldg(a.rowptr + i), end = __ldg(a.rowptr + i + 1);
                own = __ldg(sw + i);
                gather_counts<L>(a.adj, sw, beg, end, p);
                d = (int)(end - beg);
            }
            uint32_t g[L];
            cut_counts<L>(p, own, d, g);
            dsum += d;
            vc_add<L, CP>(C, g);
            if (UPDATE && VAR) {
                // Per-p-bit variability (pbit.py:57-75): act = r + tanh(lam (i0 raw + delta)).
                // +1 iff u >= t* = (1 - tanh x) / 2 = 1 / (1 + e^{2x}).  The draw's top
                // word zh (u 2^32 in [zh - 1, zh + 2)) is compared with an fp32
                // t = rcp(1 + ex2(2 log2e x)), x from fl32 lam and lam*delta:
                //   |x - x64| <= A 2^-21.9, A = |lam| |i0 raw| + |lam delta|
                //   |t - t*|  <= A 2^-22 + |x| 2^-24 + 2^-22   (ex2, rcp, 1 + E rounding)
                // so with diff = zh - t 2^32 (one rounding, <= 2^7; zh -> fp32 <= 2^7)
                // |u 2^32 - t* 2^32 - diff| < (A + 1) 2^11 + 2^9 < M = (A + 2) 2^11.
                // |diff| >= M decides; otherwise (probability ~2^-16) the update is
                // recomputed in fp64 with the libm-exact tanh, as _kernels.py:150-152.
                // (An fp16 profile halves these coalesced bytes but its wider margin
                // sends ~5e-4 of the updates to the divergent recheck: measured 10 %
                // slower here; the timing kernels, whose reads are scattered, use it.)
                const uint32_t ui = (uint32_t)i;
                const float2 *pr = a.prof + (size_t)w * 32 * a.n + i;
                const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + ch) * 1024 + lane : nullptr;
                uint32_t word = 0, exact = 0;
                uint32_t X[4];  // NATIVE: the current Philox block (trials 4k .. 4k + 3)
                auto decide = [&](int b, float2 lv) {
                    int pop = 0;
#pragma unroll
                    for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                    const int raw = 2 * pop - d;
                    const float ir = a.i0f * (float)raw;
                    uint32_t zh;
                    if (NATIVE) {  // u 2^32 = X + 1/2: the replay margin covers it
                        if ((b & 3) == 0)
                            philox4x32_10_rk(ui, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                             kNativeTagR, a.rk, X);
                        zh = X[b & 3];
                    } else if (CACHED) {
                        const uint2 v = __ldcs(ctile + b * 32);
                        zh = packed_hash_hi_y(v.x ^ count, v.y);
                    } else {
                        const uint2 kc = key[b];
                        uint32_t sl, sh;
                        packed_first_absorb(kc.x ^ ui, kc.y, sl, sh);
                        zh = packed_hash_hi(sl, sh, count);
                    }
                    const uint32_t v = var_prefilter(lv, ir, zh, a.margin);
                    if (v & 2u)
                        exact |= 1u << b;
                    else
                        word |= (v & 1u) << b;
                    if (a.inp_out)
                        a.inp_out[((size_t)w * 32 + b) * a.n + i] = __dmul_rn(a.i0, (double)raw);
                };
#pragma unroll
                for (int b = 0; b < 32; ++b) decide(b, __ldg(pr + (size_t)b * a.n));
                if (exact) word |= var_exact_bits<L, NATIVE>(a, exact, p, d, w, i, count);
                a.snew[(size_t)w * a.n + i] = word;
            } else if (UPDATE && TAPSA) {
                // S = p of this cycle + the other filled slots of the ring, in
                // SP = L + 3 planes (the host admits alpha * dmax < 2^SP)
                constexpr int SP = L + 3;
                constexpr int SB = SP < 8 ? SP : 8;  // planes carried by the byte transposition
                uint32_t S[SP];
#pragma unroll
                for (int r = 0; r < SP; ++r) S[r] = r < L ? p[r] : 0u;
                uint32_t *ring = a.ring + (size_t)w * a.alpha * L * a.n + i;
                for (int qs = 0; qs < a.filled; ++qs) {
                    if (qs == a.slot) continue;
                    uint32_t x[L];
#pragma unroll
                    for (int r = 0; r < L; ++r) x[r] = ring[(size_t)(qs * L + r) * a.n];
                    vc_add<L, SP>(S, x);
                }
#pragma unroll
                for (int r = 0; r < L; ++r) ring[(size_t)(a.slot * L + r) * a.n] = p[r];
                // byte-transpose S: B[k] byte j = S of trial 4k + j (low 8 planes; the
                // shifted copies of a 4-bit group never overlap, so the multiply is a spread)
                uint32_t B[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    B[k] = 0;
#pragma unroll
                    for (int r = 0; r < SB; ++r) {
                        const uint32_t x4 = (S[r] >> (4 * k)) & 0xFu;
                        B[k] |= (x4 * (0x00204081u << r)) & (0x01010101u << r);
                    }
                }
                // thresholds indexed by acc + f dmax = 2 S + f (dmax - d) (f = filled)
                const int off = a.filled * (a.dmax - d);
                const uint32_t rb = (uint32_t)__cvta_generic_to_shared(sthr) + 8u * (uint32_t)off;
                const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + ch) * 1024 + lane : nullptr;
                uint32_t word = 0, tie = 0xffffffffu;
                const uint32_t ui = (uint32_t)i;
                uint32_t X[4];  // NATIVE: the current Philox block
#pragma unroll
                for (int b = 31; b >= 0; --b) {
                    const int k = b >> 2, j = b & 3;
                    uint32_t sv = (B[k] >> (8 * j)) & 0xFFu;
#pragma unroll
                    for (int r = 8; r < SP; ++r) sv |= ((S[r] >> b) & 1u) << r;
                    const uint32_t addr = rb + (sv << 4);
                    uint2 t;
                    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(t.x), "=r"(t.y) : "r"(addr));
                    if (NATIVE) {
                        if ((b & 3) == 3)
                            philox4x32_10_rk(ui, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                             kNativeTagR, a.rk, X);
                        native_decide(X[b & 3], t, word);
                    } else if (CACHED) {
                        const uint2 v = __ldcs(ctile + b * 32);
                        tie = min(tie, packed_decide_y(v.x ^ count, v.y, t, word));
                    } else {
                        const uint2 kc = key[b];
                        uint32_t sl, sh;
                        packed_first_absorb(kc.x ^ ui, kc.y, sl, sh);
                        tie = min(tie, packed_second_decide(sl, sh, count, t, word));
                    }
                }
                if (!NATIVE && tie < 2) {  // rare near-tie: exact 64-bit test
                    word = 0;
                    for (int b = 0; b < 32; ++b) {
                        int sb = 0;
                        for (int r = 0; r < SP; ++r) sb |= (int)((S[r] >> b) & 1u) << r;
                        const uint64_t x1 = (a.krg[(size_t)w * 32 + b]) ^ (uint64_t)ui;
                        const uint64_t x2 = (mix64(x1) + PB_GAMMA) ^ (uint64_t)count;
                        word |= (uint32_t)hash_ge_exact(x2, a.thr[2 * sb + off]) << b;
                    }
                }
                a.snew[(size_t)w * a.n + i] = word;
                if (a.raw_out) {  // last cycle only: acc = sum of the filled raw fields
                    for (int b = 0; b < 32; ++b) {
                        int sb = 0;
                        for (int r = 0; r < SP; ++r) sb |= (int)((S[r] >> b) & 1u) << r;
                        a.raw_out[(size_t)i * a.Tp + w * 32 + b] = (int16_t)(2 * sb - a.filled * d);
                    }
                }
            } else if (UPDATE && SPSA) {
                // Stalled rule (_kernels.py:139-144): the drive is i0[c'] * raw' of the
                // p-bit's last fresh update, so its threshold is thr_all[c' * K + raw' + dmax];
                // sidx keeps that index per (trial, node).  A fresh draw refreshes it unless
                // u = u01(key, TAG_STALL, i, count) < p_stall; the first update is always fresh.
                uint32_t *sidx = a.sidx + (size_t)w * 32 * a.n + i;
                const int base = a.cycle * a.Kc + a.dmax - d;      // fresh index = base + 2 pop
                const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + ch) * 1024 + lane : nullptr;
                const uint32_t ui = (uint32_t)i;
                // pass 1: stall bits of the 32 trials (exactly, before any index is replaced)
                uint32_t stallw = 0;
                if (NATIVE && a.cycle > 0) {
                    // stall iff X_stall < S (p_stall64 = S = ceil(p 2^32 - 1/2), u = (X + 1/2) 2^-32)
                    const uint64_t ns = (1ULL << 32) - a.p_stall64;
                    const uint2 pst = make_uint2((uint32_t)ns, (uint32_t)(ns >> 32));
                    uint32_t gew = 0, Xs[4];
#pragma unroll
                    for (int b = 31; b >= 0; --b) {
                        if ((b & 3) == 3)
                            philox4x32_10_rk(ui, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                             kNativeTagStall, a.rk, Xs);
                        native_decide(Xs[b & 3], pst, gew);
                    }
                    stallw = ~gew;
                } else if (a.cycle > 0) {
                    const uint2 pst = make_uint2(~(uint32_t)(a.p_stall64 >> 32),
                                                 (uint32_t)(a.p_stall64 >> 32));
                    uint32_t gew = 0, ties = 0xffffffffu;
                    const uint2 *keys = skeys + wib * 32;
#pragma unroll 8
                    for (int b = 31; b >= 0; --b) {
                        const uint2 ks = keys[b];
                        uint32_t sl, sh;
                        packed_first_absorb(ks.x ^ ui, ks.y, sl, sh);
                        ties = min(ties, packed_second_decide(sl, sh, count, pst, gew));
                    }
                    stallw = ~gew;  // H_stall < p_stall64 -> stall
                    if (ties < 2) {
                        stallw = 0;
                        for (int b = 0; b < 32; ++b) {
                            const uint64_t xs = (a.kst[(size_t)w * 32 + b]) ^ (uint64_t)ui;
                            const uint64_t xs2 = (mix64(xs) + PB_GAMMA) ^ (uint64_t)count;
                            stallw |= (uint32_t)!hash_ge_exact(xs2, a.p_stall64) << b;
                        }
                    }
                }
                // pass 2: drive (stalled: the stored index, a coalesced load, then
                // its threshold's high word from the all-cycles table; fresh: this
                // cycle's shared-memory table, and the index is stored), then the
                // activation decision.  Eight trials per group: the stalled trials'
                // loads are issued together before the group's decisions.
                uint32_t word = 0, tie = 0xffffffffu;
                uint32_t X[4];  // NATIVE: the current Philox block of the activation draws
                // groups of GS trials (native: 4, its stalled drives need both threshold words)
                constexpr int GS = NATIVE ? 4 : 8;
                for (int gq = 32 / GS - 1; gq >= 0; --gq) {
                    uint32_t th[GS], keep[GS];
#pragma unroll
                    for (int j = GS - 1; j >= 0; --j) {
                        const int b = gq * GS + j;
                        th[j] = ((stallw >> b) & 1u) ? sidx[(size_t)b * a.n] : 0u;
                        keep[j] = th[j];
                    }
                    uint32_t tlo[GS];  // NATIVE: low words of 2^32 - T of the stalled drives
#pragma unroll
                    for (int j = GS - 1; j >= 0; --j) {
                        const int b = gq * GS + j;
                        if ((stallw >> b) & 1u) {
                            if (NATIVE) {
                                const uint64_t nt = (1ULL << 32) - __ldg(a.thr_all + th[j]);
                                tlo[j] = (uint32_t)nt;
                                th[j] = (uint32_t)(nt >> 32);
                            } else {
                                th[j] = __ldg(a.thr_hi_all + th[j]);
                            }
                        }
                    }
#pragma unroll
                    for (int j = GS - 1; j >= 0; --j) {
                        const int b = gq * GS + j;
                        int pop = 0;
#pragma unroll
                        for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                        uint2 t;
                        uint32_t nidx = keep[j];
                        if ((stallw >> b) & 1u) {
                            t = NATIVE ? make_uint2(tlo[j], th[j]) : make_uint2(~th[j], th[j]);
                        } else {
                            t = NIB ? sthr[d * 16 + pop] : sthr[2 * pop - d + a.dmax];
                            nidx = (uint32_t)(base + 2 * pop);
                        }
                        // every lane stores (stalled p-bits their unchanged index): whole
                        // sectors, no partial-sector read-modify-write in L2 / HBM
                        if (a.sidx_full) sidx[(size_t)b * a.n] = nidx;
                        else if (!((stallw >> b) & 1u)) sidx[(size_t)b * a.n] = nidx;
                        if (NATIVE) {
                            if ((b & 3) == 3)
                                philox4x32_10_rk(ui, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                                 kNativeTagR, a.rk, X);
                            native_decide(X[b & 3], t, word);
                        } else if (CACHED) {
                            const uint2 v = __ldcs(ctile + b * 32);
                            tie = min(tie, packed_decide_y(v.x ^ count, v.y, t, word));
                        } else {
                            const uint2 kc = key[b];
                            uint32_t sl, sh;
                            packed_first_absorb(kc.x ^ ui, kc.y, sl, sh);
                            tie = min(tie, packed_second_decide(sl, sh, count, t, word));
                        }
                    }
                }
                if (!NATIVE && tie < 2) {  // rare near-tie in an activation draw: exact 64-bit test
                    word = 0;
                    for (int b = 0; b < 32; ++b) {
                        const uint32_t idx = sidx[(size_t)b * a.n];
                        const uint64_t x1 = (a.krg[(size_t)w * 32 + b]) ^ (uint64_t)ui;
                        const uint64_t x2 = (mix64(x1) + PB_GAMMA) ^ (uint64_t)count;
                        word |= (uint32_t)hash_ge_exact(x2, a.thr_all[idx]) << b;
                    }
                }
                a.snew[(size_t)w * a.n + i] = word;
            } else if (UPDATE) {
                const uint2 *tb = sthr + (a.dmax - d);   // entry for raw = 2 pop - d
                // cache tile of (word w, chunk ch): [b][lane], so trial b of this
                // lane sits at a compile-time offset b * 256 B
                const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + ch) * 1024 + lane : nullptr;
                uint32_t word = 0, tie = 0xffffffffu;
                const uint32_t ui = (uint32_t)i;
                uint32_t X[4];  // NATIVE: the current Philox block (trials 4k .. 4k + 3)
                // NIB: transpose the L count planes into 32 nibbles (N[k] nibble j =
                // count of trial 8k + j), a few ops per 32 trials instead of 2L per trial
                uint32_t N[4] = {0u, 0u, 0u, 0u};
                uint32_t rb = 0;
                if (NIB) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
#pragma unroll
                        for (int r = 0; r < L; ++r) {
                            uint32_t x = (p[r] >> (8 * k)) & 0xFFu;
                            x = (x | (x << 12)) & 0x000F000Fu;
                            x = (x | (x << 6)) & 0x03030303u;
                            x = (x | (x << 3)) & 0x11111111u;
                            N[k] |= x << r;
                        }
                    }
                    rb = (uint32_t)__cvta_generic_to_shared(sthr) + (uint32_t)d * 128u;
                }
#pragma unroll
                for (int b = 31; b >= 0; --b) {
                    uint2 t;
                    if (NIB) {
                        const int k = b >> 3, j = b & 7;
                        const uint32_t x = j == 0 ? (N[k] << 3) : (N[k] >> (4 * j - 3));
                        const uint32_t addr = (x & 0x78u) | rb;
                        asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(t.x), "=r"(t.y) : "r"(addr));
                    } else {
                        int pop = 0;
#pragma unroll
                        for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                        t = tb[2 * pop];
                    }
                    if (NATIVE) {
                        // one Philox call per four trials: counter (i, count, group, tag)
                        if ((b & 3) == 3)
                            philox4x32_10_rk(ui, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                             kNativeTagR, a.rk, X);
                        uint32_t dummy;
                        asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
                            : "=r"(dummy), "=r"(word) : "r"(X[b & 3]), "r"(t.x), "r"(word), "r"(word + t.y));
                    } else if (CACHED) {
                        const uint2 v = __ldcs(ctile + b * 32);
                        tie = min(tie, packed_decide_n2(v.x ^ count, v.y, t, word));
                    } else {
                        const uint2 kc = key[b];
                        uint32_t sl, sh;
                        packed_first_absorb(kc.x ^ ui, kc.y, sl, sh);
                        tie = min(tie, packed_second_decide_n2(sl, sh, count, t, word));
                    }
                }
                if (!NATIVE && tie < 3) {  // rare: some trial's draw is within 1 of its threshold -> exact 64-bit test
                    word = 0;
                    for (int b = 0; b < 32; ++b) {
                        int pop = 0;
                        for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                        const uint64_t x1 = (a.krg[(size_t)w * 32 + b]) ^ (uint64_t)ui;
                        const uint64_t x2 = (mix64(x1) + PB_GAMMA) ^ (uint64_t)count;
                        word |= (uint32_t)hash_ge_exact(x2, a.thr[2 * pop - d + a.dmax]) << b;
                    }
                }
                a.snew[(size_t)w * a.n + i] = word;
                if (a.raw_out) {  // last cycle only: the raw field each trial's update used
                    for (int b = 0; b < 32; ++b) {
                        int pop = 0;
                        for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                        a.raw_out[(size_t)i * a.Tp + w * 32 + b] = (int16_t)(2 * pop - d);
                    }
                }
            }
        }
    }
    warp_cut_flush(C, dsum, lane, live ? a.pacc + (size_t)w * 32 : nullptr);
}

// ------------------------------------------- packed sweep with a timing spread
// Per-p-bit periods (pbit.py:74) gate each trial: in sub-step `count` only the
// trials whose period divides it fire (_kernels.py:126), typically ~15 %, and
// unevenly across the lanes of a warp.  The fire mask of a (word, node) comes
// from the bit-sliced periods: OR over the present periods dividing `count`
// (host list) of the AND of the matching plane polarities.  The warp then
// compacts its fired (lane, trial) pairs into a shared-memory list and deals
// them round-robin to its 32 lanes, so a launch costs ~max(mean fires, 1)
// decisions per lane instead of the maximum lane's count; results return
// through shared-memory bit masks.  Decision and exact recheck as ALG=3.
constexpr int kMaxDivisors = 256;
constexpr size_t kTimingSmem = kPackedWarps * 32 * sizeof(uint2) + kMaxDivisors * 8 * 4 +
                               2 * kPackedWarps * 32 * 4 + kPackedWarps * 1024 * 4;

template <int L, bool NATIVE = false>
__global__ void __launch_bounds__(kPackedThreads, PBSA_PACKED_MIN_BLOCKS)
    packed_sweep_timing(PackedArgs a) {
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ unsigned long long smem_u64[];
    uint2 *skey = reinterpret_cast<uint2 *>(smem_u64);                           // [warps][32]
    uint32_t *sdivx = reinterpret_cast<uint32_t *>(skey + kPackedWarps * 32);    // [div][8]
    uint32_t *sres = sdivx + kMaxDivisors * 8;                                   // [warps][32]
    uint32_t *sexm = sres + kPackedWarps * 32;                                   // [warps][32]
    uint32_t *sfl = sexm + kPackedWarps * 32;                                    // [warps][1024]
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gwarp = blockIdx.x * kPackedWarps + wib;
    const int w = gwarp / a.warps_per_word;
    const int q = gwarp % a.warps_per_word;
    const bool live = w < a.W;
    uint2 *key = skey + wib * 32;
    key[lane] = live ? a.kfc[(size_t)w * 32 + lane] : make_uint2(0, 0);
    // per divisor and plane: 0 selects the plane, ~0 its complement (planes
    // above nplanes are zero, so their complement passes)
    for (int k = threadIdx.x; k < a.ndiv * 8; k += blockDim.x) {
        const uint32_t pv = a.divs[k >> 3];
        const int pl = k & 7;
        sdivx[k] = (pl < a.nplanes && ((pv >> pl) & 1u)) ? 0u : 0xffffffffu;
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t count = a.count;
    constexpr int CP = CutPlanes<L>::value;
    uint32_t C[CP];
#pragma unroll
    for (int r = 0; r < CP; ++r) C[r] = 0;
    int dsum = 0;
    uint32_t *fl = sfl + wib * 1024, *res = sres + wib * 32, *exm = sexm + wib * 32;

    if (live) {
        const uint32_t *sw = a.sold + (size_t)w * a.n;
        for (int ch = q; ch < a.chunks; ch += a.warps_per_word) {
            const int i = ch * 32 + lane;
            const bool valid = i < a.n;
            // (the gather is issued with the period planes: with a timing
            // spread almost every warp has some firing trial)
            uint32_t own = 0, fire = 0, beg = 0, end = 0;
            uint32_t pl[8];
            const bool reg4 = L >= 3 && a.reg4;
            if (valid) {
                if (!reg4) {
                    beg = __ldg(a.rowptr + i);
                    end = __ldg(a.rowptr + i + 1);
                }
                own = __ldg(sw + i);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
                pl[k] = (valid && k < a.nplanes) ? __ldg(a.pplanes + ((size_t)w * a.nplanes + k) * a.n + i) : 0u;
            uint32_t p[L];
            int d = (int)(end - beg);
            if (reg4) {
                if (valid) {
                    gather_counts_reg4<L>(a.adj, sw, i, p);
                    d = 4;
                } else {
#pragma unroll
                    for (int r = 0; r < L; ++r) p[r] = 0;
                }
            } else {
                gather_counts<L>(a.adj, sw, beg, end, p);
            }
            if (valid) {
                for (int dv = 0; dv < a.ndiv; ++dv) {
                    const uint4 x0 = *reinterpret_cast<const uint4 *>(sdivx + dv * 8);
                    const uint4 x1 = *reinterpret_cast<const uint4 *>(sdivx + dv * 8 + 4);
                    fire |= (pl[0] ^ x0.x) & (pl[1] ^ x0.y) & (pl[2] ^ x0.z) & (pl[3] ^ x0.w) &
                            (pl[4] ^ x1.x) & (pl[5] ^ x1.y) & (pl[6] ^ x1.z) & (pl[7] ^ x1.w);
                }
            }
            if (a.do_cut && valid) {
                uint32_t g[L];
                cut_counts<L>(p, own, d, g);
                dsum += d;
                vc_add<L, CP>(C, g);
            }
            // compact the warp's fired (lane, trial) pairs with their raw fields
            const int c = __popc(fire);
            int off = c;
#pragma unroll
            for (int sft = 1; sft < 32; sft <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, off, sft);
                if (lane >= sft) off += v;
            }
            const int F = __shfl_sync(0xffffffffu, off, 31);
            off -= c;
            for (uint32_t f = fire; f; f &= f - 1) {
                const int b = __ffs(f) - 1;
                int pop = 0;
#pragma unroll
                for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                fl[off++] = ((uint32_t)(2 * pop - d + 1024) << 10) | ((uint32_t)lane << 5) | (uint32_t)b;
            }
            res[lane] = 0;
            exm[lane] = 0;
            __syncwarp();
            // two list entries per lane and round, their profile loads in flight together
            auto fire_one = [&](uint32_t e, __half2 lv) {
                const int b = (int)(e & 31u), l = (int)((e >> 5) & 31u), raw = (int)(e >> 10) - 1024;
                const int ii = ch * 32 + l;
                const float ir = a.i0f * (float)raw;
                uint32_t zh;
                if (NATIVE) {  // one Philox block per fired trial (fired trials are sparse)
                    uint32_t o[4];
                    philox4x32_10_rk((uint32_t)ii, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                     kNativeTagR, a.rk, o);
                    zh = (b & 2) ? ((b & 1) ? o[3] : o[2]) : ((b & 1) ? o[1] : o[0]);
                } else {
                    const uint2 kc = key[b];
                    uint32_t sl, sh;
                    packed_first_absorb(kc.x ^ (uint32_t)ii, kc.y, sl, sh);
                    zh = packed_hash_hi(sl, sh, count);
                }
                const uint32_t v = var_prefilter(lv, ir, zh, a.margin);
                if (v & 2u)
                    atomicOr(exm + l, 1u << b);
                else if (v & 1u)
                    atomicOr(res + l, 1u << b);
                if (a.inp_out) a.inp_out[((size_t)w * 32 + b) * a.n + ii] = __dmul_rn(a.i0, (double)raw);
            };
            auto prof_of = [&](uint32_t e) {
                return __ldg(a.prof16 + ((size_t)w * a.n + ch * 32 + ((e >> 5) & 31u)) * 32 + (e & 31u));
            };
            // four list entries per lane and round, their profile loads in flight together
            for (int k = lane; k < F; k += 128) {
                uint32_t e[4];
                __half2 lv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) e[j] = k + 32 * j < F ? fl[k + 32 * j] : fl[k];
#pragma unroll
                for (int j = 0; j < 4; ++j) lv[j] = prof_of(e[j]);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (k + 32 * j < F) fire_one(e[j], lv[j]);
            }
            __syncwarp();
            if (valid) {
                uint32_t word = (own & ~fire) | res[lane];
                const uint32_t ex = exm[lane];
                if (ex) word |= var_exact_bits<L, NATIVE>(a, ex, p, d, w, i, count);
                a.snew[(size_t)w * a.n + i] = word;
            }
            __syncwarp();
        }
    }
    warp_cut_flush(C, dsum, lane, live ? a.pacc + (size_t)w * 32 : nullptr);
}

// ------------------------------------------------ resident multi-cycle sweep
// For words whose whole spin state fits shared memory (8 n bytes double
// buffered, n <= ~25k), one thread-block cluster anneals one trial word for
// ALL cycles in a single launch: every CTA keeps a full copy of the word's
// state in shared memory, updates its slice of the nodes (gather from local
// shared memory, the packed kernel's decision), and writes each new word into
// its own and every peer CTA's next buffer through distributed shared memory;
// one cluster barrier per cycle is the synchronous commit of _kernels.py:151-155.
// No per-cycle launches and no state traffic through L2 -- the lever for
// small graphs and batches, where per-cycle launch latency dominates.
struct ResidentArgs {
    const uint32_t *s_in;       // [W][n] initial words
    uint32_t *s_out;            // [W][n] final words
    const uint32_t *rowptr;     // [n+1]
    const uint32_t *adj;        // [nnz] column | (J < 0) << 31
    const uint2 *kfc;           // [Tp] folded per-trial constants
    const uint2 *acache;        // [W][chunks][32][32] first-absorb cache, or null
    const uint64_t *krg;        // [Tp] absorb(key, TAG_R) + GAMMA
    const uint64_t *thr;        // [cycles][K] thresholds
    unsigned long long *pacc;   // [cycles+1][Tp]
    int16_t *raw_out;           // [n][Tp] raw fields of the last cycle
    int n, W, Tp, K, dmax, chunks, cycles, t_res;
    // VARU: per-p-bit lam/delta without a timing spread (ALG=3 decision)
    const float2 *prof;         // [Tp][n] {fl32(lam), fl32(lam * delta)}
    const double *lam64, *del64;
    const double *i0;           // [cycles]
    double *inp_out;            // [Tp][n] inputs of the last cycle
    float margin;
    // NATIVE: Philox draws (philox.cuh); thr then holds the 32-bit thresholds
    uint32_t rk[20];            // round keys of the native seed
    uint32_t ngroup;            // Philox trial group of word 0: (first trial) / 4
    // TAPSA: the time-averaged rule; the CTA's slice of the bit-sliced ring
    // lives in shared memory and is written back to ring at the end
    uint32_t *ring;             // [W][alpha][L][n]
    int alpha;
};

constexpr int kResidentExtraPlanes = 3;  // cut counters for up to 32 nodes per thread

template <int L, bool CACHED, bool VARU = false, bool NATIVE = false, bool TAPSA = false>
__global__ void __launch_bounds__(512, 1) resident_sweep(ResidentArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int w = (int)(blockIdx.x / CS);
    constexpr bool NIB = L <= 4 && !VARU && !TAPSA;
    extern __shared__ unsigned long long smem_u64[];
    uint2 *sthrA = reinterpret_cast<uint2 *>((reinterpret_cast<uintptr_t>(smem_u64) + 511) & ~(uintptr_t)511);
    const int tab_entries = VARU ? 0 : (NIB && !TAPSA) ? (a.dmax + 1) * 16 : a.K;
    // two threshold tables: cycle c reads one while cycle c + 1's entries, loaded
    // at the start of cycle c, are written into the other (the table load's L2
    // latency leaves the per-cycle critical path; (dmax + 1) 16 entries keep
    // the second table 128-byte aligned for the NIB address trick)
    uint2 *sthrB = sthrA + tab_entries;
    uint2 *key = sthrB + tab_entries;
    uint32_t *S0 = reinterpret_cast<uint32_t *>(key + 32);
    uint32_t *S1 = S0 + a.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int k = tid; k < a.n; k += blockDim.x) S0[k] = a.s_in[(size_t)w * a.n + k];
    if (tid < 32) key[tid] = a.kfc[(size_t)w * 32 + tid];
    const int per = (a.n + CS - 1) / CS;
    const int lo = rank * per, hi = min(a.n, lo + per);
    // this CTA's nodes' CSR rows in shared memory too (a cluster barrier
    // flushes L1, which would otherwise re-fetch them from L2 every cycle)
    uint32_t *ringS = S1 + a.n;                 // TAPSA: [alpha][L][per] bit-sliced counts
    uint32_t *rowS = ringS + (TAPSA ? a.alpha * L * per : 0);  // [hi - lo + 1], relative offsets
    uint32_t *adjS = rowS + (per + 1);          // [rowptr[hi] - rowptr[lo]]
    const uint32_t r0 = a.rowptr[lo], r1 = a.rowptr[hi];
    for (int k = tid; k <= hi - lo; k += blockDim.x) rowS[k] = a.rowptr[lo + k] - r0;
    for (uint32_t k = tid; k < r1 - r0; k += blockDim.x) adjS[k] = a.adj[r0 + k];
    uint32_t *cs = S0, *ns = S1;
    constexpr int CP = L + 2 + kResidentExtraPlanes;
    // table entry k of a cycle: its source in the cycle's threshold row (-1: unused)
    // and its shared-memory form
    auto tab_src = [&](int k) -> int {
        if (TAPSA) return k;  // [acc + f dmax]
        if (NIB) {
            const int d = k >> 4, pp = k & 15;
            return pp <= d ? 2 * pp - d + a.dmax : -1;
        }
        return k;
    };
    auto tab_entry = [&](uint64_t tfull) -> uint2 {
        const uint32_t thi = (uint32_t)(tfull >> 32);
        if (TAPSA) {  // replay (~thi, thi) (packed_decide_y); native 2^32 - T
            const uint64_t nt = (1ULL << 32) - tfull;
            return NATIVE ? make_uint2((uint32_t)nt, (uint32_t)(nt >> 32)) : make_uint2(~thi, thi);
        }
        // replay: the 33-bit ~thi + 2 (packed_decide_n2); native: 2^32 - T
        const uint64_t n2 = NATIVE ? (1ULL << 32) - tfull : (uint64_t)(~thi) + 2u;
        return make_uint2((uint32_t)n2, (uint32_t)(n2 >> 32));
    };
    for (int k = tid; k < tab_entries; k += blockDim.x) {
        const int sidx = tab_src(k);
        sthrA[k] = tab_entry(sidx >= 0 ? a.thr[sidx] : 0ULL);
    }
    cluster.sync();  // every CTA of the cluster runs before any shared-memory exchange

    // next-cycle entries held in registers per thread (the rest load at the cycle's
    // end; measured: the replayed plain rule is 4 % faster without the registers)
    constexpr int kPre = VARU ? 0 : TAPSA ? 4 : NATIVE ? 2 : 0;
    for (int c = 0; c <= a.cycles; ++c) {
        const int cc = c < a.cycles ? c : a.cycles - 1;
        const uint64_t *thr = a.thr + (size_t)cc * a.K;
        uint2 *sthr = (c & 1) ? sthrB : sthrA;
        uint2 *sthr_next = (c & 1) ? sthrA : sthrB;
        const bool pre = c + 1 < a.cycles;
        uint64_t pv[kPre > 0 ? kPre : 1];
#pragma unroll
        for (int j = 0; j < kPre; ++j) {
            const int k = tid + j * (int)blockDim.x;
            const int sidx = k < tab_entries ? tab_src(k) : -1;
            pv[j] = (pre && sidx >= 0) ? __ldg(thr + a.K + sidx) : 0ULL;
        }
        const uint32_t count = (uint32_t)(c * a.t_res);
        const uint32_t grp = a.ngroup + 8u * (uint32_t)w;  // NATIVE: Philox group of trial 0
        uint32_t C[CP];
#pragma unroll
        for (int r = 0; r < CP; ++r) C[r] = 0;
        int dsum = 0;
        for (int base = lo + warp * 32; base < hi; base += nwarps * 32) {
            const int i = base + lane;
            if (i >= hi) continue;
            const uint32_t beg = rowS[i - lo], end = rowS[i - lo + 1];
            const uint32_t own = cs[i];
            uint32_t p[L];
            count_neighbours<L>(beg, end, [&](uint32_t k) {
                const uint32_t e = adjS[k];
                return cs[e & 0x7fffffffu] ^ (uint32_t)((int32_t)e >> 31);
            }, p);
            const int d = (int)(end - beg);
            uint32_t g[L];
            cut_counts<L>(p, own, d, g);
            dsum += d;
            vc_add<L, CP>(C, g);
            if (c == a.cycles) continue;  // final cut pass
            const uint32_t ui = (uint32_t)i;
            const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + (i >> 5)) * 1024 + (i & 31) : nullptr;
            if (VARU) {  // the packed ALG=3 decision (sigmoid prefilter, exact recheck)
                const double i0 = a.i0[cc];
                const float i0f = (float)i0;
                const float2 *pr = a.prof + (size_t)w * 32 * a.n + i;
                uint32_t word = 0, exact = 0;
                uint32_t X[4];
#pragma unroll
                for (int b = 0; b < 32; ++b) {
                    int pop = 0;
#pragma unroll
                    for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                    const int raw = 2 * pop - d;
                    const float2 lv = __ldg(pr + (size_t)b * a.n);
                    const float ir = i0f * (float)raw;
                    uint32_t zh;
                    if (NATIVE) {
                        if ((b & 3) == 0)
                            philox4x32_10_rk(ui, count, grp + (uint32_t)(b >> 2), kNativeTagR, a.rk, X);
                        zh = X[b & 3];
                    } else if (CACHED) {
                        const uint2 v = __ldcs(ctile + b * 32);
                        zh = packed_hash_hi_y(v.x ^ count, v.y);
                    } else {
                        const uint2 kc = key[b];
                        uint32_t sl, sh;
                        packed_first_absorb(kc.x ^ ui, kc.y, sl, sh);
                        zh = packed_hash_hi(sl, sh, count);
                    }
                    const uint32_t v = var_prefilter(lv, ir, zh, a.margin);
                    if (v & 2u)
                        exact |= 1u << b;
                    else
                        word |= (v & 1u) << b;
                    if (a.inp_out && c == a.cycles - 1)
                        a.inp_out[((size_t)w * 32 + b) * a.n + i] = __dmul_rn(i0, (double)raw);
                }
                while (exact) {
                    const int b = __ffs(exact) - 1;
                    exact &= exact - 1;
                    int pop = 0;
                    for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                    const size_t idx = ((size_t)w * 32 + b) * a.n + i;
                    double r;
                    if (NATIVE) {
                        uint32_t o[4];
                        philox4x32_10_rk(ui, count, grp + (uint32_t)(b >> 2), kNativeTagR, a.rk, o);
                        const uint32_t x = (b & 2) ? ((b & 1) ? o[3] : o[2]) : ((b & 1) ? o[1] : o[0]);
                        r = __dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(2.0, (double)x), 1.0), 0x1p-32), 1.0);
                    } else {
                        const uint64_t x1 = (a.krg[(size_t)w * 32 + b]) ^ (uint64_t)ui;
                        const uint64_t x2 = (mix64(x1) + PB_GAMMA) ^ (uint64_t)count;
                        r = __dsub_rn(__dmul_rn(2.0, u01_of(mix64(x2))), 1.0);
                    }
                    const double xx = __dmul_rn(a.lam64[idx], __dadd_rn(__dmul_rn(i0, (double)(2 * pop - d)),
                                                                       a.del64[idx]));
                    word |= (uint32_t)(__dadd_rn(r, pb_libm_tanh(xx)) >= 0.0) << b;
                }
                ns[i] = word;
                for (int r = 1; r < CS; ++r) {
                    const int peer = rank + r < CS ? rank + r : rank + r - CS;
                    *cluster.map_shared_rank(ns + i, peer) = word;
                }
                continue;
            }
            if (TAPSA) {
                // time-averaged rule (_kernels.py:131-138), as packed_sweep ALG=1:
                // S = this cycle's count + the other filled ring slots (SP planes),
                // thresholds indexed by acc + f dmax = 2 S + f (dmax - d)
                constexpr int SP = L + 3;
                constexpr int SB = SP < 8 ? SP : 8;
                const int filled = min(c + 1, a.alpha), slot = c % a.alpha;
                uint32_t S[SP];
#pragma unroll
                for (int r = 0; r < SP; ++r) S[r] = r < L ? p[r] : 0u;
                uint32_t *rg = ringS + (i - lo);
                for (int qs = 0; qs < filled; ++qs) {
                    if (qs == slot) continue;
                    uint32_t x[L];
#pragma unroll
                    for (int r = 0; r < L; ++r) x[r] = rg[(qs * L + r) * per];
                    vc_add<L, SP>(S, x);
                }
#pragma unroll
                for (int r = 0; r < L; ++r) rg[(slot * L + r) * per] = p[r];
                uint32_t B[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    B[k] = 0;
#pragma unroll
                    for (int r = 0; r < SB; ++r) {
                        const uint32_t x4 = (S[r] >> (4 * k)) & 0xFu;
                        B[k] |= (x4 * (0x00204081u << r)) & (0x01010101u << r);
                    }
                }
                const int off = filled * (a.dmax - d);
                const uint32_t rb = (uint32_t)__cvta_generic_to_shared(sthr) + 8u * (uint32_t)off;
                uint32_t word = 0, tie = 0xffffffffu;
                uint32_t X[4];
#pragma unroll
                for (int b = 31; b >= 0; --b) {
                    const int k = b >> 2, j = b & 3;
                    uint32_t sv = (B[k] >> (8 * j)) & 0xFFu;
#pragma unroll
                    for (int r = 8; r < SP; ++r) sv |= ((S[r] >> b) & 1u) << r;
                    const uint32_t addr = rb + (sv << 4);
                    uint2 t;
                    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(t.x), "=r"(t.y) : "r"(addr));
                    if (NATIVE) {
                        if ((b & 3) == 3)
                            philox4x32_10_rk(ui, count, grp + (uint32_t)(b >> 2), kNativeTagR, a.rk, X);
                        native_decide(X[b & 3], t, word);
                    } else if (CACHED) {
                        const uint2 v = __ldcs(ctile + b * 32);
                        tie = min(tie, packed_decide_y(v.x ^ count, v.y, t, word));
                    } else {
                        const uint2 kc = key[b];
                        uint32_t sl, sh;
                        packed_first_absorb(kc.x ^ ui, kc.y, sl, sh);
                        tie = min(tie, packed_second_decide(sl, sh, count, t, word));
                    }
                }
                if (!NATIVE && tie < 2) {  // rare near-tie: exact 64-bit test
                    word = 0;
                    for (int b = 0; b < 32; ++b) {
                        int sb = 0;
                        for (int r = 0; r < SP; ++r) sb |= (int)((S[r] >> b) & 1u) << r;
                        const uint64_t x1 = (a.krg[(size_t)w * 32 + b]) ^ (uint64_t)ui;
                        const uint64_t x2 = (mix64(x1) + PB_GAMMA) ^ (uint64_t)count;
                        word |= (uint32_t)hash_ge_exact(x2, thr[2 * sb + off]) << b;
                    }
                }
                ns[i] = word;
                for (int r = 1; r < CS; ++r) {
                    const int peer = rank + r < CS ? rank + r : rank + r - CS;
                    *cluster.map_shared_rank(ns + i, peer) = word;
                }
                if (a.raw_out && c == a.cycles - 1) {  // acc = sum of the filled raw fields
                    for (int b = 0; b < 32; ++b) {
                        int sb = 0;
                        for (int r = 0; r < SP; ++r) sb |= (int)((S[r] >> b) & 1u) << r;
                        a.raw_out[(size_t)i * a.Tp + w * 32 + b] = (int16_t)(2 * sb - filled * d);
                    }
                }
                continue;
            }
            uint32_t word = 0, tie = 0xffffffffu;
            uint32_t N[4] = {0u, 0u, 0u, 0u};
            uint32_t rb = 0;
            if (NIB) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
#pragma unroll
                    for (int r = 0; r < L; ++r) {
                        uint32_t x = (p[r] >> (8 * k)) & 0xFFu;
                        x = (x | (x << 12)) & 0x000F000Fu;
                        x = (x | (x << 6)) & 0x03030303u;
                        x = (x | (x << 3)) & 0x11111111u;
                        N[k] |= x << r;
                    }
                }
                rb = (uint32_t)__cvta_generic_to_shared(sthr) + (uint32_t)d * 128u;
            }
            const uint2 *tb = sthr + (a.dmax - d);
            uint32_t X[4];
#pragma unroll
            for (int b = 31; b >= 0; --b) {
                uint2 t;
                if (NIB) {
                    const int k = b >> 3, j = b & 7;
                    const uint32_t x = j == 0 ? (N[k] << 3) : (N[k] >> (4 * j - 3));
                    const uint32_t addr = (x & 0x78u) | rb;
                    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(t.x), "=r"(t.y) : "r"(addr));
                } else {
                    int pop = 0;
#pragma unroll
                    for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                    t = tb[2 * pop];
                }
                if (NATIVE) {
                    if ((b & 3) == 3)
                        philox4x32_10_rk(ui, count, grp + (uint32_t)(b >> 2), kNativeTagR, a.rk, X);
                    uint32_t dummy;
                    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
                        : "=r"(dummy), "=r"(word) : "r"(X[b & 3]), "r"(t.x), "r"(word), "r"(word + t.y));
                } else if (CACHED) {
                    const uint2 v = __ldcs(ctile + b * 32);
                    tie = min(tie, packed_decide_n2(v.x ^ count, v.y, t, word));
                } else {
                    const uint2 kc = key[b];
                    uint32_t sl, sh;
                    packed_first_absorb(kc.x ^ ui, kc.y, sl, sh);
                    tie = min(tie, packed_second_decide_n2(sl, sh, count, t, word));
                }
            }
            if (!NATIVE && tie < 3) {  // rare: a draw within 1 of its threshold -> exact 64-bit test
                word = 0;
                for (int b = 0; b < 32; ++b) {
                    int pop = 0;
                    for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                    const uint64_t x1 = (a.krg[(size_t)w * 32 + b]) ^ (uint64_t)ui;
                    const uint64_t x2 = (mix64(x1) + PB_GAMMA) ^ (uint64_t)count;
                    word |= (uint32_t)hash_ge_exact(x2, thr[2 * pop - d + a.dmax]) << b;
                }
            }
            ns[i] = word;
            for (int r = 1; r < CS; ++r) {  // the peers' copies of this word
                const int peer = rank + r < CS ? rank + r : rank + r - CS;
                *cluster.map_shared_rank(ns + i, peer) = word;
            }
            if (a.raw_out && c == a.cycles - 1) {
                for (int b = 0; b < 32; ++b) {
                    int pop = 0;
                    for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                    a.raw_out[(size_t)i * a.Tp + w * 32 + b] = (int16_t)(2 * pop - d);
                }
            }
        }
        warp_cut_flush(C, dsum, lane, a.pacc + (size_t)c * a.Tp + (size_t)w * 32);
        if (pre) {  // next cycle's table (its readers, cycle c - 1, passed the last barrier)
#pragma unroll
            for (int j = 0; j < kPre; ++j) {
                const int k = tid + j * (int)blockDim.x;
                if (k < tab_entries) sthr_next[k] = tab_entry(pv[j]);
            }
            for (int k = tid + kPre * (int)blockDim.x; k < tab_entries; k += blockDim.x) {
                const int sidx = tab_src(k);
                sthr_next[k] = tab_entry(sidx >= 0 ? thr[a.K + sidx] : 0ULL);
            }
        }
        if (c < a.cycles) {
            cluster.sync();  // every copy of the next state (and table) is complete
            uint32_t *t = cs;
            cs = ns;
            ns = t;
        }
    }
    if (TAPSA) {  // the ring slots written in the run, for the history output
        const int slots = min(a.cycles, a.alpha);
        for (int k = tid; k < slots * L * (hi - lo); k += blockDim.x) {
            const int j = k % (hi - lo), qr = k / (hi - lo);
            a.ring[((size_t)w * a.alpha * L + qr) * a.n + lo + j] = ringS[qr * per + j];
        }
    }
    for (int i = lo + tid; i < hi; i += blockDim.x) a.s_out[(size_t)w * a.n + i] = cs[i];
}

// Resident variant of the timing-spread kernel (packed_sweep_timing): one
// cluster per trial word runs every sub-step of the run in one launch, the
// word's state, CSR slice and bit-sliced periods in shared memory, one
// cluster barrier per sub-step.  With ten sub-steps per cycle the launched
// form is bound by launch latency on small graphs; this removes it.
struct RLaunch {
    uint32_t count;
    int cycle, do_cut, ndiv, div_off, inp;
    double i0;
};

struct ResidentTimingArgs {
    const uint32_t *s_in;
    uint32_t *s_out;
    const uint32_t *rowptr, *adj;
    const uint2 *kfc;
    const uint64_t *krg;
    const __half2 *prof;        // [W][n][32] fp16 pairs (node-major: a node's 32 trials contiguous)
    const double *lam64, *del64;
    const uint32_t *pplanes;    // [W][nplanes][n]
    const uint8_t *divs;
    const RLaunch *launches;
    int nlaunch;
    const double *i0;           // [cycles]
    unsigned long long *pacc;   // [cycles+1][Tp]
    double *inp_out;            // [Tp][n]
    int n, W, Tp, nplanes, cycles;
    float margin;
    uint32_t rk[20];            // NATIVE: Philox round keys
    uint32_t ngroup;            // NATIVE: Philox trial group of word 0
    int prof_smem;              // the CTA's profile slice is staged in shared memory
    int split;                  // 16 nodes per warp, two lanes per node
};

template <int L, bool NATIVE = false>
__global__ void __launch_bounds__(512, 1) resident_timing(ResidentTimingArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int w = (int)(blockIdx.x / CS);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int per = (a.n + CS - 1) / CS;
    const int lo = rank * per, hi = min(a.n, lo + per);
    extern __shared__ unsigned long long smem_u64[];
    uint2 *key = reinterpret_cast<uint2 *>(smem_u64);        // [32]
    uint32_t *S0 = reinterpret_cast<uint32_t *>(key + 32);   // [n]
    uint32_t *S1 = S0 + a.n;                                  // [n]
    uint32_t *res = S1 + a.n;                                 // [nwarps][32]
    uint32_t *exm = res + nwarps * 32;                        // [nwarps][32]
    uint32_t *fl = exm + nwarps * 32;                         // [nwarps][1024]
    uint32_t *sdivx = fl + nwarps * 1024;                     // [kMaxDivisors][8]
    uint32_t *plS = sdivx + kMaxDivisors * 8;                 // [nplanes][per]
    // the CTA's slice of the fp16 profile ([per][32], node-major) when it fits:
    // fired p-bits then read it at shared-memory latency instead of L2's
    __half2 *profS = reinterpret_cast<__half2 *>(plS + a.nplanes * per);
    uint32_t *rowS = reinterpret_cast<uint32_t *>(profS + (a.prof_smem ? per * 32 : 0));  // [per + 1]
    uint32_t *adjS = rowS + per + 1;
    for (int k = tid; k < a.n; k += blockDim.x) S0[k] = a.s_in[(size_t)w * a.n + k];
    if (tid < 32) key[tid] = a.kfc[(size_t)w * 32 + tid];
    const uint32_t r0 = a.rowptr[lo], r1 = a.rowptr[hi];
    for (int k = tid; k <= hi - lo; k += blockDim.x) rowS[k] = a.rowptr[lo + k] - r0;
    for (uint32_t k = tid; k < r1 - r0; k += blockDim.x) adjS[k] = a.adj[r0 + k];
    for (int k = tid; k < a.nplanes * per; k += blockDim.x) {
        const int pl = k / per, j = k - pl * per;
        plS[k] = lo + j < hi ? a.pplanes[((size_t)w * a.nplanes + pl) * a.n + lo + j] : 0u;
    }
    if (a.prof_smem) {
        const __half2 *src = a.prof + ((size_t)w * a.n + lo) * 32;
        for (int k = tid; k < (hi - lo) * 32; k += blockDim.x) profS[k] = src[k];
    }
    uint32_t *cs = S0, *ns = S1;
    uint32_t *wfl = fl + warp * 1024, *wres = res + warp * 32, *wexm = exm + warp * 32;
    constexpr int CP = L + 2 + kResidentExtraPlanes;
    uint32_t C[CP];
#pragma unroll
    for (int r = 0; r < CP; ++r) C[r] = 0;
    int dsum = 0;
    cluster.sync();

    RLaunch Rn = a.launches[0];
    for (int li = 0; li < a.nlaunch; ++li) {
        const RLaunch R = Rn;
        if (li + 1 < a.nlaunch) Rn = a.launches[li + 1];  // in flight during this sub-step
        const bool update = R.cycle < a.cycles;
        const double i0 = R.i0;
        const float i0f = (float)i0;
        const uint32_t count = R.count;
        // this sub-step's dividing periods as plane polarity masks (0 selects the
        // plane, ~0 its complement; absent planes are zero and pass)
        for (int k = tid; k < R.ndiv * 8; k += blockDim.x) {
            const uint32_t pv = a.divs[R.div_off + (k >> 3)];
            const int pl = k & 7;
            sdivx[k] = (pl < a.nplanes && ((pv >> pl) & 1u)) ? 0u : 0xffffffffu;
        }
        __syncthreads();
        // split mode (a.split): a warp takes 16 nodes, lanes l and l + 16 share
        // node base + l and split its neighbour list and its fired trials (half
        // the per-warp critical path of a 32-node chunk; the sub-step is
        // latency-bound at ~2 warps per scheduler).  Otherwise lane = node.
        const int cw = a.split ? 16 : 32;
        for (int base = lo + warp * cw; base < hi; base += nwarps * cw) {
            const int hl = a.split ? lane & 15 : lane, half = a.split ? lane >> 4 : 0;
            const int i = base + hl;
            const bool valid = i < hi;
            uint32_t own = 0, fire = 0, beg = 0, end = 0;
            if (valid) {
                own = cs[i];
                beg = rowS[i - lo];
                end = rowS[i - lo + 1];
                if (update) {
                    uint32_t pl[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) pl[k] = k < a.nplanes ? plS[k * per + (i - lo)] : 0u;
                    for (int dv = 0; dv < R.ndiv; ++dv) {
                        const uint4 x0 = *reinterpret_cast<const uint4 *>(sdivx + dv * 8);
                        const uint4 x1 = *reinterpret_cast<const uint4 *>(sdivx + dv * 8 + 4);
                        fire |= (pl[0] ^ x0.x) & (pl[1] ^ x0.y) & (pl[2] ^ x0.z) & (pl[3] ^ x0.w) &
                                (pl[4] ^ x1.x) & (pl[5] ^ x1.y) & (pl[6] ^ x1.z) & (pl[7] ^ x1.w);
                    }
                }
            }
            const bool any = __any_sync(0xffffffffu, fire != 0);
            if (!R.do_cut && !any) {  // nothing fires: carry the words
                if (valid && update && half == 0) {
                    ns[i] = own;
                    for (int r = 1; r < CS; ++r)
                        *cluster.map_shared_rank(ns + i, rank + r < CS ? rank + r : rank + r - CS) = own;
                }
                continue;
            }
            uint32_t p[L];
            const uint32_t mid = a.split ? beg + ((end - beg + 1) >> 1) : end;
            count_neighbours<L>(half ? mid : beg, half ? end : mid, [&](uint32_t k) {
                const uint32_t e = adjS[k];
                return cs[e & 0x7fffffffu] ^ (uint32_t)((int32_t)e >> 31);
            }, p);
            if (a.split) {   // the two halves' partial counts, added bit-sliced (the sum is <= d < 2^L)
                uint32_t carry = 0;
#pragma unroll
                for (int r = 0; r < L; ++r) {
                    const uint32_t q = __shfl_xor_sync(0xffffffffu, p[r], 16);
                    const uint32_t sm = p[r] ^ q ^ carry;
                    carry = (p[r] & q) | (carry & (p[r] ^ q));
                    p[r] = sm;
                }
            }
            const int d = (int)(end - beg);
            if (R.do_cut && valid && half == 0) {
                uint32_t g[L];
                cut_counts<L>(p, own, d, g);
                dsum += d;
                vc_add<L, CP>(C, g);
            }
            if (!update) continue;
            // warp-balanced fired (lane, trial, raw) list, as packed_sweep_timing
            const uint32_t myfire = a.split ? fire & (half ? 0xffff0000u : 0x0000ffffu) : fire;
            const int c = __popc(myfire);
            int off = c;
#pragma unroll
            for (int sft = 1; sft < 32; sft <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, off, sft);
                if (lane >= sft) off += v;
            }
            const int F = __shfl_sync(0xffffffffu, off, 31);
            off -= c;
            for (uint32_t f = myfire; f; f &= f - 1) {
                const int b = __ffs(f) - 1;
                int pop = 0;
#pragma unroll
                for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                wfl[off++] = ((uint32_t)(2 * pop - d + 1024) << 10) | ((uint32_t)hl << 5) | (uint32_t)b;
            }
            if (lane < cw) {
                wres[lane] = 0;
                wexm[lane] = 0;
            }
            __syncwarp();
            // two list entries per lane and round, their profile loads in flight together
            auto fire_one = [&](uint32_t e, __half2 lv) {
                const int b = (int)(e & 31u), l = (int)((e >> 5) & 31u), raw = (int)(e >> 10) - 1024;
                const int ii = base + l;
                const float ir = i0f * (float)raw;
                uint32_t zh;
                if (NATIVE) {
                    uint32_t o[4];
                    philox4x32_10_rk((uint32_t)ii, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                     kNativeTagR, a.rk, o);
                    zh = (b & 2) ? ((b & 1) ? o[3] : o[2]) : ((b & 1) ? o[1] : o[0]);
                } else {
                    const uint2 kc = key[b];
                    uint32_t sl, sh;
                    packed_first_absorb(kc.x ^ (uint32_t)ii, kc.y, sl, sh);
                    zh = packed_hash_hi(sl, sh, count);
                }
                const uint32_t v = var_prefilter(lv, ir, zh, a.margin);
                if (v & 2u)
                    atomicOr(wexm + l, 1u << b);
                else if (v & 1u)
                    atomicOr(wres + l, 1u << b);
                if (R.inp) a.inp_out[((size_t)w * 32 + b) * a.n + ii] = __dmul_rn(i0, (double)raw);
            };
            auto prof_of = [&](uint32_t e) {
                const int j = base + (int)((e >> 5) & 31u);
                return a.prof_smem ? profS[(j - lo) * 32 + (int)(e & 31u)]
                                   : __ldg(a.prof + ((size_t)w * a.n + j) * 32 + (e & 31u));
            };
            for (int k = lane; k < F; k += 64) {
                const uint32_t e0 = wfl[k];
                const bool two = k + 32 < F;
                const uint32_t e1 = two ? wfl[k + 32] : e0;
                const __half2 lv0 = prof_of(e0), lv1 = prof_of(e1);
                fire_one(e0, lv0);
                if (two) fire_one(e1, lv1);
            }
            __syncwarp();
            if (valid && half == 0) {
                uint32_t word = (own & ~fire) | wres[hl];
                uint32_t ex = wexm[hl];
                while (ex) {  // rare near-tie: the reference's fp64 arithmetic
                    const int b = __ffs(ex) - 1;
                    ex &= ex - 1;
                    int pop = 0;
                    for (int r = 0; r < L; ++r) pop |= (int)((p[r] >> b) & 1u) << r;
                    const size_t idx = ((size_t)w * 32 + b) * a.n + i;
                    double r;
                    if (NATIVE) {
                        uint32_t o[4];
                        philox4x32_10_rk((uint32_t)i, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                         kNativeTagR, a.rk, o);
                        const uint32_t x = (b & 2) ? ((b & 1) ? o[3] : o[2]) : ((b & 1) ? o[1] : o[0]);
                        r = __dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(2.0, (double)x), 1.0), 0x1p-32), 1.0);
                    } else {
                        const uint64_t x1 = (a.krg[(size_t)w * 32 + b]) ^ (uint64_t)(uint32_t)i;
                        const uint64_t x2 = (mix64(x1) + PB_GAMMA) ^ (uint64_t)count;
                        r = __dsub_rn(__dmul_rn(2.0, u01_of(mix64(x2))), 1.0);
                    }
                    const double xx = __dmul_rn(a.lam64[idx], __dadd_rn(__dmul_rn(i0, (double)(2 * pop - d)),
                                                                       a.del64[idx]));
                    word |= (uint32_t)(__dadd_rn(r, pb_libm_tanh(xx)) >= 0.0) << b;
                }
                ns[i] = word;
                for (int r = 1; r < CS; ++r)
                    *cluster.map_shared_rank(ns + i, rank + r < CS ? rank + r : rank + r - CS) = word;
            }
            __syncwarp();
        }
        if (R.do_cut) {
            warp_cut_flush(C, dsum, lane, a.pacc + (size_t)R.cycle * a.Tp + (size_t)w * 32);
#pragma unroll
            for (int r = 0; r < CP; ++r) C[r] = 0;
            dsum = 0;
        }
        if (update) {
            cluster.sync();
            uint32_t *t = cs;
            cs = ns;
            ns = t;
        }
    }
    for (int i = lo + tid; i < hi; i += blockDim.x) a.s_out[(size_t)w * a.n + i] = cs[i];
}

// Packed spins [W][n] -> int8 [T][n]
__global__ void unpack_spins(const uint32_t *__restrict__ s, int8_t *__restrict__ out, int n,
                             int W, int T) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)n * T) return;
    const int t = (int)(g / n), i = (int)(g % n);
    out[g] = ((s[(size_t)(t >> 5) * n + i] >> (t & 31)) & 1u) ? 1 : -1;
}

// inputs[t][i] = i0_last * (acc_last[i][t] / filled): the last drive of the
// plain rule (filled = 1, acc = raw; _kernels.py:146) or the time-averaged
// rule (_kernels.py:138); raw_last is the packed kernel's last-cycle output.
__global__ void inputs_from_raw(const int16_t *__restrict__ raw, double *__restrict__ out,
                                double i0_last, int n, int Tp, int T, double filled) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)n * T) return;
    const int t = (int)(g / n), i = (int)(g % n);
    out[g] = __dmul_rn(i0_last, __ddiv_rn((double)raw[(size_t)i * Tp + t], filled));
}

// SpSA last drive inputs[t][i] = i0[c'] * raw' from the packed drive index
// c' * K + raw' + dmax (_kernels.py:144, 147).
__global__ void inputs_from_sidx(const uint32_t *__restrict__ sidx, const double *__restrict__ i0,
                                 double *__restrict__ out, int n, int T, int K, int dmax) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)n * T) return;
    const int t = (int)(g / n), i = (int)(g % n);
    const uint32_t idx = sidx[(size_t)t * n + i];  // [W][32][n] == [trial][n]
    const int c = (int)(idx / (uint32_t)K), raw = (int)(idx % (uint32_t)K) - dmax;
    out[g] = __dmul_rn(i0[c], (double)raw);
}

// TApSA history output [T][n][alpha] from the packed ring: slot q holds the
// raw field 2p - d of the last cycle that wrote it (0.0 if never written).
template <int L>
__global__ void hist_from_ring(const uint32_t *__restrict__ ring, const uint32_t *__restrict__ rowptr,
                               int n, int T, int alpha, int written, double *__restrict__ out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)n * T) return;
    const int t = (int)(g / n), i = (int)(g % n);
    const int w = t >> 5, b = t & 31;
    const int d = (int)(rowptr[i + 1] - rowptr[i]);
    for (int q = 0; q < alpha; ++q) {
        double v = 0.0;
        if (q < written) {
            int p = 0;
            for (int r = 0; r < L; ++r)
                p |= (int)((ring[((size_t)(w * alpha + q) * L + r) * n + i] >> b) & 1u) << r;
            v = (double)(2 * p - d);
        }
        out[g * alpha + q] = v;
    }
}

// ----------------------------------------------------------- general path
struct GeneralArgs {
    const int8_t *sold;
    int8_t *snew;
    const uint32_t *rowptr;
    const uint32_t *col;
    const double *val;
    const double *h;
    const double *lam;     // [n][Tp] or [n] (shared) or null (1.0)
    const double *delta;   // same layout, null = 0.0
    const int32_t *period; // same layout, null = t_res
    int shared_profile;
    double *inputs;        // [n][Tp]
    int32_t *counts;       // [n][Tp]
    double *hist;          // [n][alpha][Tp] (TAPSA only)
    const uint64_t *kr;    // [Tp] absorb(key, TAG_R)
    const uint64_t *kst;   // [Tp] absorb(key, TAG_STALL)
    int n, Tp, T, algo, alpha, t_res;
    double i0, p_stall;
    uint32_t count;
};

__global__ void __launch_bounds__(256) general_substep(GeneralArgs a) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)a.n * a.Tp) return;
    const int i = (int)(g / a.Tp), t = (int)(g % a.Tp);
    const int8_t cur = a.sold[g];
    const int64_t pidx = a.shared_profile ? i : g;
    const uint32_t per = a.period ? (uint32_t)a.period[pidx] : (uint32_t)a.t_res;
    if (t >= a.T || a.count % per != 0) {
        a.snew[g] = cur;
        return;
    }
    // raw = h_i + sum_k values[k] * spins[indices[k]], CSR order (_kernels.py:128-130)
    double raw = a.h[i];
    const uint32_t beg = a.rowptr[i], end = a.rowptr[i + 1];
    for (uint32_t k = beg; k < end; ++k)
        raw = __dadd_rn(raw, __dmul_rn(a.val[k], (double)a.sold[(size_t)a.col[k] * a.Tp + t]));
    const int32_t cnt = a.counts[g];
    double inp;
    if (a.algo == 1) {  // TAPSA (_kernels.py:131-138)
        const size_t base = (size_t)i * a.alpha;
        a.hist[(base + cnt % a.alpha) * a.Tp + t] = raw;
        const int filled = cnt + 1 < a.alpha ? cnt + 1 : a.alpha;
        double acc = 0.0;
        for (int q = 0; q < filled; ++q) acc = __dadd_rn(acc, a.hist[(base + q) * a.Tp + t]);
        inp = __dmul_rn(a.i0, __ddiv_rn(acc, (double)filled));
    } else if (a.algo == 2) {  // SPSA (_kernels.py:139-144)
        if (cnt == 0) {
            inp = __dmul_rn(a.i0, raw);
        } else {
            const double u = u01_of(absorb(absorb(a.kst[t], (uint64_t)i), (uint64_t)a.count));
            inp = u < a.p_stall ? a.inputs[g] : __dmul_rn(a.i0, raw);
        }
    } else {
        inp = __dmul_rn(a.i0, raw);
    }
    a.inputs[g] = inp;
    a.counts[g] = cnt + 1;
    const double lam = a.lam ? a.lam[pidx] : 1.0;
    const double del = a.delta ? a.delta[pidx] : 0.0;
    const double r = __dsub_rn(__dmul_rn(2.0, u01_of(absorb(absorb(a.kr[t], (uint64_t)i),
                                                            (uint64_t)a.count))), 1.0);
    const double act = __dadd_rn(r, pb_libm_tanh(__dmul_rn(lam, __dadd_rn(inp, del))));
    a.snew[g] = act >= 0.0 ? 1 : -1;
}

// ------------------------------------------------- general path, active lists
// For integer-valued models (every MAX-CUT instance) the sub-step touches only
// the p-bits that fire: (trial, node) pairs are bucketed by update period on
// the host, and a sub-step with counter `count` processes the concatenation of
// the buckets whose period divides it (descriptors {start, cum, len}).  One
// thread per firing p-bit; the local field is an exact integer sum (equal to
// the reference's fp64 CSR-order sum because every partial sum is an integer
// below 2^53).  New spins are staged and scattered by a second kernel, which
// keeps the synchronous snapshot semantics of _kernels.py:151-155.
struct ActiveArgs {
    const int8_t *s;          // [n][Tp]
    uint32_t *st_g;           // staged pair index
    int8_t *st_v;             // staged new spin
    const uint32_t *list;     // all (node << tshift | trial) entries, bucketed by period
    const int4 *desc;         // [ndesc] {start in list, cumulative offset, length, 0}
    int ndesc, total;
    const uint32_t *rowptr, *col;
    const int32_t *vali;      // integer couplings, CSR order
    const int32_t *hi;        // integer fields or null
    const double *lam, *delta;
    int shared_profile;
    double *inputs;           // [Np] list order
    int32_t *counts;          // [Np] list order
    int32_t *hist;            // [alpha][Np] raw fields (TAPSA), list order
    int64_t Np;               // list length (= trials * n)
    const uint64_t *kr, *kst;
    const uint64_t *thr;      // [K] this cycle's thresholds (table mode) or null
    int rawmin;
    int tshift;
    uint32_t tmask;
    int Tp, alpha, algo;
    double i0, p_stall;
    uint32_t count;
};

constexpr int kMaxActiveDesc = 512;

__global__ void __launch_bounds__(256) general_active(ActiveArgs a) {
    __shared__ int4 sdesc[kMaxActiveDesc];
    for (int k = threadIdx.x; k < a.ndesc; k += blockDim.x) sdesc[k] = a.desc[k];
    __syncthreads();
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= a.total) return;
    int lo = 0, hi = a.ndesc - 1;  // last descriptor with cum <= pos
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sdesc[mid].y <= pos) lo = mid; else hi = mid - 1;
    }
    // per-p-bit state lives in list order: a firing p-bit always sits at the
    // same list position, so state loads/stores of a launch are coalesced
    const uint32_t li = (uint32_t)(sdesc[lo].x + (pos - sdesc[lo].y));
    const uint32_t e = a.list[li];
    const int i = (int)(e >> a.tshift), t = (int)(e & a.tmask);
    const size_t g = (size_t)i * a.Tp + t;
    int raw = a.hi ? a.hi[i] : 0;
    const uint32_t beg = a.rowptr[i], end = a.rowptr[i + 1];
    for (uint32_t k = beg; k < end; ++k) raw += a.vali[k] * (int)a.s[(size_t)a.col[k] * a.Tp + t];
    const int32_t cnt = a.counts[li];
    double inp;
    if (a.algo == 1) {  // TAPSA (_kernels.py:131-138); integer partial sums are exact in fp64
        int32_t *ring = a.hist + li;
        ring[(size_t)(cnt % a.alpha) * a.Np] = raw;
        const int filled = cnt + 1 < a.alpha ? cnt + 1 : a.alpha;
        long long acc = 0;
        for (int q = 0; q < filled; ++q) acc += ring[(size_t)q * a.Np];
        inp = __dmul_rn(a.i0, __ddiv_rn((double)acc, (double)filled));
    } else if (a.algo == 2 && cnt > 0) {  // SPSA (_kernels.py:139-144)
        const double u = u01_of(absorb(absorb(a.kst[t], (uint64_t)i), (uint64_t)a.count));
        inp = u < a.p_stall ? a.inputs[li] : __dmul_rn(a.i0, (double)raw);
    } else {
        inp = __dmul_rn(a.i0, (double)raw);
    }
    a.inputs[li] = inp;
    a.counts[li] = cnt + 1;
    const uint64_t h = absorb(absorb(a.kr[t], (uint64_t)i), (uint64_t)a.count);
    bool up;
    if (a.thr) {  // lam = 1, delta = 0, plain rule: exact integer threshold per (cycle, raw)
        const uint64_t thr = a.thr[raw - a.rawmin];
        up = h >= thr && thr != ~0ULL;
    } else {
        double x = inp;
        if (a.lam) {
            const size_t pidx = a.shared_profile ? (size_t)i : (size_t)li;
            x = __dmul_rn(a.lam[pidx], __dadd_rn(inp, a.delta[pidx]));
        }
        const double r = __dsub_rn(__dmul_rn(2.0, u01_of(h)), 1.0);
        // Prefilter with single-precision tanhf (<= 2 ulp) of x rounded to
        // float: |tanhf((float)x) - tanh(x)| < 2^-21 for every x, so whenever
        // |r + tanhf| >= 2^-16 the sign equals the sign of r + libm tanh(x).
        // Only the rare near-ties evaluate the libm-exact fp64 tanh.
        const double sres = __dadd_rn(r, (double)tanhf(__double2float_rn(x)));
        if (fabs(sres) >= 0x1p-16)
            up = sres >= 0.0;
        else
            up = __dadd_rn(r, pb_libm_tanh(x)) >= 0.0;
    }
    a.st_g[pos] = (uint32_t)g;
    a.st_v[pos] = up ? 1 : -1;
}

// ---------------------------------------- active lists, plain rule, fast path
// The plain rule (pSA; SpSA with p = 0) with a timing spread: only the
// firing p-bits of a sub-step cost work (active lists as above), and the
// rule keeps no per-p-bit state -- the update count of a firing p-bit is
// count / period and its input is i0 * raw -- so a launch reads the list,
// the fp32 profile pair (list order, coalesced) and the int8 neighbour spins,
// and writes only the flips (compacted per warp) plus, during the last
// p_max sub-steps, the inputs.  The draw uses the folded per-trial constants
// of the packed path; the decision is the packed variability kernel's
// sigmoid prefilter with its exact fp64 recheck, or the exact integer
// threshold table when lam = 1 and delta = 0.
struct FastArgs {
    int8_t *s;                // [n][Tp] spins (read-only in the launch)
    const uint32_t *list;     // (node << tshift | trial), bucketed by period
    const int4 *desc;         // [ndesc] {start, cumulative offset, length, 0}
    int ndesc, total;
    const uint32_t *rowptr, *col;
    const int32_t *vali, *hi; // integer couplings (CSR order), integer fields or null
    const float2 *prof;       // [Np] list order, or [n] shared; null: table mode
    const double *lam64, *del64;
    int shared_profile;
    const uint64_t *thr;      // [K] this cycle's thresholds (table mode) or null
    int rawmin;
    const uint2 *kfc;         // [Tp] folded per-trial constants of absorb(key, TAG_R)
    const uint64_t *krg;      // [Tp] absorb(key, TAG_R) + GAMMA
    int tshift;
    uint32_t tmask;
    int Tp;
    uint32_t count;
    double i0;
    float i0f, margin;
    double *inputs;           // [Np] list order (last p_max sub-steps) or null
    uint32_t *flips;          // compacted spin indices to negate
    uint32_t *nflips;         // this launch's flip counter
};

__global__ void __launch_bounds__(256) active_fast(FastArgs a) {
    __shared__ int4 sdesc[kMaxActiveDesc];
    for (int k = threadIdx.x; k < a.ndesc; k += blockDim.x) sdesc[k] = a.desc[k];
    __syncthreads();
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    bool flip = false;
    uint32_t g = 0;
    if (pos < a.total) {
        int lo = 0, hi = a.ndesc - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sdesc[mid].y <= pos) lo = mid; else hi = mid - 1;
        }
        const uint32_t li = (uint32_t)(sdesc[lo].x + (pos - sdesc[lo].y));
        const uint32_t e = __ldg(a.list + li);
        const int i = (int)(e >> a.tshift), t = (int)(e & a.tmask);
        g = (uint32_t)i * (uint32_t)a.Tp + (uint32_t)t;
        int raw = a.hi ? __ldg(a.hi + i) : 0;
        const uint32_t beg = __ldg(a.rowptr + i), end = __ldg(a.rowptr + i + 1);
        for (uint32_t k = beg; k < end; ++k)
            raw += __ldg(a.vali + k) * (int)a.s[(size_t)__ldg(a.col + k) * a.Tp + t];
        const uint2 kc = __ldg(a.kfc + t);
        uint32_t sl, sh;
        packed_first_absorb(kc.x ^ (uint32_t)i, kc.y, sl, sh);
        bool up, exact = false;
        if (a.thr) {  // lam = 1, delta = 0: H >= thr exactly
            const uint64_t thr = __ldg(a.thr + (raw - a.rawmin));
            const uint32_t zh = packed_hash_hi(sl, sh, a.count);
            const uint32_t thi = (uint32_t)(thr >> 32);
            // top words decide unless they (nearly) tie
            up = zh > thi;
            exact = zh - thi + 1u <= 2u;  // |zh - thi| <= 1
        } else {
            const float2 lv = __ldg(a.prof + (a.shared_profile ? (size_t)i : (size_t)li));
            const float ir = a.i0f * (float)raw;
            const float x = fmaf(lv.x, ir, lv.y);
            const float A = fmaf(fabsf(lv.x), fabsf(ir), fabsf(lv.y));
            const float tt = rcp_approx(1.0f + ex2_approx(x * 2.88539008f));
            const uint32_t zh = packed_hash_hi(sl, sh, a.count);
            const float diff = fmaf(-tt, 4294967296.0f, __uint2float_rn(zh));
            up = diff > 0.0f;
            exact = fabsf(diff) < fmaf(A, 2048.0f * a.margin, 4096.0f * a.margin);
        }
        if (exact) {  // the reference's arithmetic on the full 64-bit draw
            const uint64_t x1 = __ldg(a.krg + t) ^ (uint64_t)(uint32_t)i;
            const uint64_t H = mix64((mix64(x1) + PB_GAMMA) ^ (uint64_t)a.count);
            if (a.thr) {
                const uint64_t thr = __ldg(a.thr + (raw - a.rawmin));
                up = H >= thr && thr != ~0ULL;
            } else {
                const size_t pidx = a.shared_profile ? (size_t)i : (size_t)li;
                const double r = __dsub_rn(__dmul_rn(2.0, u01_of(H)), 1.0);
                const double xx = __dmul_rn(a.lam64[pidx], __dadd_rn(__dmul_rn(a.i0, (double)raw), a.del64[pidx]));
                up = __dadd_rn(r, pb_libm_tanh(xx)) >= 0.0;
            }
        }
        if (a.inputs) a.inputs[li] = __dmul_rn(a.i0, (double)raw);
        flip = up != (a.s[g] > 0);
    }
    // warp-aggregated compaction of the flips
    const unsigned m = __ballot_sync(0xffffffffu, flip);
    if (m) {
        const int lane = threadIdx.x & 31;
        uint32_t base = 0;
        if (lane == __ffs(m) - 1) base = atomicAdd(a.nflips, (uint32_t)__popc(m));
        base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
        if (flip) a.flips[base + __popc(m & ((1u << lane) - 1u))] = g;
    }
}

// negate the spins flipped by one sub-step (grid sized for the launch's firings)
__global__ void apply_flips(int8_t *__restrict__ s, const uint32_t *__restrict__ flips,
                            const uint32_t *__restrict__ nflips) {
    const uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos < *nflips) {
        const uint32_t g = flips[pos];
        s[g] = (int8_t)-s[g];
    }
}

// list-order per-p-bit state -> [trial][node][k] output rows
template <typename TS, typename TD>
__global__ void list_to_trial_major(const TS *__restrict__ src, const uint32_t *__restrict__ list,
                                    int64_t Np, int tshift, uint32_t tmask, int n, int K,
                                    TD *__restrict__ dst) {
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= Np) return;
    const uint32_t e = list[li];
    const int64_t row = (int64_t)(e & tmask) * n + (e >> tshift);
    for (int k = 0; k < K; ++k) dst[row * K + k] = (TD)src[(size_t)k * Np + li];
}

__global__ void general_scatter(int8_t *__restrict__ s, const uint32_t *__restrict__ st_g,
                                const int8_t *__restrict__ st_v, int total) {
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos < total) s[st_g[pos]] = st_v[pos];
}

__global__ void widen_hist(const int32_t *__restrict__ src, double *__restrict__ dst, int64_t n) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) dst[g] = (double)src[g];
}

// Per-cycle cut and integer energy over edges, spins int8 [n][Tp].
// grid.x chunks the edge range, threads cover trials.
struct StatsArgs {
    const int8_t *s;
    const uint32_t *ge_i, *ge_j;
    const int64_t *ge_w;
    const uint32_t *me_i, *me_j;
    const int64_t *me_wi;   // integer couplings (int_energy mode)
    const int64_t *hi;      // integer fields (int_energy mode), null if all zero
    int64_t gm, mm;
    int n, Tp, T;
    int chunks;
    unsigned long long *cut_acc;   // [Tp] for this cycle
    unsigned long long *e_acc;     // [Tp] for this cycle (sum_e J s s + sum_i h s)
};

__global__ void general_stats(StatsArgs a) {
    const int t = blockIdx.y * blockDim.x + threadIdx.x;
    if (t >= a.T) return;
    const int ch = blockIdx.x;
    long long cut = 0, e = 0;
    {
        const int64_t per = (a.gm + a.chunks - 1) / a.chunks;
        const int64_t lo = ch * per, hi = min(a.gm, lo + per);
        for (int64_t k = lo; k < hi; ++k)
            if (a.s[(size_t)a.ge_i[k] * a.Tp + t] != a.s[(size_t)a.ge_j[k] * a.Tp + t])
                cut += a.ge_w[k];
    }
    if (a.e_acc) {
        const int64_t per = (a.mm + a.chunks - 1) / a.chunks;
        const int64_t lo = ch * per, hi = min(a.mm, lo + per);
        for (int64_t k = lo; k < hi; ++k)
            e += a.me_wi[k] * (long long)(a.s[(size_t)a.me_i[k] * a.Tp + t] *
                                          a.s[(size_t)a.me_j[k] * a.Tp + t]);
        if (a.hi) {
            const int64_t pn = (a.n + a.chunks - 1) / a.chunks;
            const int64_t lo2 = ch * pn, hi2 = min((int64_t)a.n, lo2 + pn);
            for (int64_t i = lo2; i < hi2; ++i) e += a.hi[i] * (long long)a.s[(size_t)i * a.Tp + t];
        }
    }
    if (cut) atomicAdd(a.cut_acc + t, (unsigned long long)cut);
    if (a.e_acc && e) atomicAdd(a.e_acc + t, (unsigned long long)e);
}

// Per-trial sum over an edge list of w_e [s_a != s_b], spins int8 [n][Tp]
// read four trials per 32-bit word.  Unit weights accumulate in packed bytes
// (flushed every 255 edges); other weights per byte.  Used per cycle for the
// cut (graph weights) and, when the model is not the graph's MAX-CUT mapping,
// for sum_e J_e [s_a != s_b] (energy = sum J - 2 * that).
__global__ void differ_count(const int8_t *__restrict__ s, const uint32_t *__restrict__ ei,
                             const uint32_t *__restrict__ ej, const int32_t *__restrict__ w,
                             int64_t m, int Tq, int chunks, unsigned long long *__restrict__ out) {
    const int q = blockIdx.y * blockDim.x + threadIdx.x;
    if (q >= Tq) return;
    const uint32_t *s32 = reinterpret_cast<const uint32_t *>(s);
    const int64_t per = (m + chunks - 1) / chunks;
    const int64_t lo = blockIdx.x * per, hi = min(m, lo + per);
    long long c[4] = {0, 0, 0, 0};
    uint32_t accP = 0, accN = 0;
    int k = 0;
    for (int64_t e = lo; e < hi; ++e) {
        const uint32_t d = ((s32[(size_t)ei[e] * Tq + q] ^ s32[(size_t)ej[e] * Tq + q]) >> 1) & 0x01010101u;
        const int wv = w[e];
        if (wv == 1) {
            accP += d;
        } else if (wv == -1) {
            accN += d;
        } else {
#pragma unroll
            for (int b = 0; b < 4; ++b) c[b] += (long long)wv * ((d >> (8 * b)) & 1u);
        }
        if (++k == 255) {
#pragma unroll
            for (int b = 0; b < 4; ++b)
                c[b] += (long long)((accP >> (8 * b)) & 0xFFu) - (long long)((accN >> (8 * b)) & 0xFFu);
            accP = accN = 0;
            k = 0;
        }
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        c[b] += (long long)((accP >> (8 * b)) & 0xFFu) - (long long)((accN >> (8 * b)) & 0xFFu);
        if (c[b]) atomicAdd(out + 4 * q + b, (unsigned long long)c[b]);
    }
}

// Exact fp64 energy in the reference's sequential order (_kernels.py:157-161),
// one thread per trial; used only when couplings/fields are not integers.
__global__ void general_energy_f64(const int8_t *__restrict__ s, const double *__restrict__ h,
                                   const uint32_t *__restrict__ me_i,
                                   const uint32_t *__restrict__ me_j,
                                   const double *__restrict__ me_w, int64_t mm, int n, int Tp,
                                   int T, double *__restrict__ e_out /* [Tp] this cycle */) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    double e = 0.0;
    for (int i = 0; i < n; ++i)
        e = __dsub_rn(e, __dmul_rn(h[i], (double)s[(size_t)i * Tp + t]));
    for (int64_t k = 0; k < mm; ++k)
        e = __dsub_rn(e, __dmul_rn(__dmul_rn(me_w[k], (double)s[(size_t)me_i[k] * Tp + t]),
                                   (double)s[(size_t)me_j[k] * Tp + t]));
    e_out[t] = e;
}

// ---------------------------------------------------------------- finalise
// Per (trial, cycle): trace_cut, trace_energy from the accumulators, [T][C].
//   mode 0 (packed):  P = pacc[c+1][t]: cut = (2W + P)/4, E = -P/2
//   mode 1 (general, integer energy): cut = cut_acc[c][t], E = -e_acc[c][t]
//   mode 2 (general, fp64 energy):    cut = cut_acc[c][t], E = e_f64[c][t]
struct FinalArgs {
    const unsigned long long *pacc;
    const unsigned long long *cut_acc;
    const unsigned long long *e_acc;   // mode 1: sum_i h_i s_i, or null
    const unsigned long long *dj_acc;  // mode 1, model != graph: sum_e J [s_a != s_b]
    const double *e_f64;
    int64_t total_w;
    int64_t sum_j;
    int graph_is_model;
    int mode, has_graph;
    int C, Tp, T;
    int64_t *trace_cut;     // [T][C]
    double *trace_energy;   // [T][C]
    int64_t *best;          // [T]
};

__global__ void finalize_traces(FinalArgs a) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.T) return;
    long long best = -(1LL << 62);
    for (int c = 0; c < a.C; ++c) {
        long long cut;
        double e;
        if (a.mode == 0) {
            const long long P = (long long)a.pacc[(size_t)(c + 1) * a.Tp + t];
            cut = a.has_graph ? (2 * a.total_w + P) / 4 : 0;
            e = (double)(-(P / 2));
        } else {
            const size_t at = (size_t)c * a.Tp + t;
            cut = a.has_graph ? (long long)a.cut_acc[at] : 0;
            if (a.mode == 1) {  // integer energy: sum J s s + sum h s, from differ counts
                long long es = a.sum_j + (a.graph_is_model ? 2 * cut : -2 * (long long)a.dj_acc[at]);
                if (a.e_acc) es += (long long)a.e_acc[at];
                e = (double)(-es);
            } else {
                e = a.e_f64[at];
            }
        }
        a.trace_cut[(size_t)t * a.C + c] = cut;
        a.trace_energy[(size_t)t * a.C + c] = e;
        if (cut > best) best = cut;
    }
    a.best[t] = best;
}

__global__ void widen_i32(const int32_t *__restrict__ src, int64_t *__restrict__ dst, int64_t n) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) dst[g] = src[g];
}

// Generic tiled transpose: src [R][Cc] -> dst [Cc_used][R] (first Cc_used columns)
template <typename T>
__global__ void transpose_tile(const T *__restrict__ src, T *__restrict__ dst, int R, int Cc,
                               int Cc_used) {
    __shared__ T tile[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = r0 + y, c = c0 + threadIdx.x;
        if (r < R && c < Cc_used) tile[y][threadIdx.x] = src[(size_t)r * Cc + c];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int c = c0 + y, r = r0 + threadIdx.x;
        if (c < Cc_used && r < R) dst[(size_t)c * R + r] = tile[threadIdx.x][y];
    }
}

// Debug: device hash and tanh on arbitrary inputs.
__global__ void debug_stream(int64_t cnt, const uint64_t *key, const uint64_t *tag,
                             const uint64_t *x, const uint64_t *y, uint64_t *out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < cnt) out[g] = absorb(absorb(absorb(key[g], tag[g]), x[g]), y[g]);
}

__global__ void debug_philox(int64_t cnt, const uint32_t *ctr, const uint32_t *key, uint32_t *out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    uint32_t o[4];
    philox4x32_10(ctr[4 * k], ctr[4 * k + 1], ctr[4 * k + 2], ctr[4 * k + 3], key[2 * k],
                  key[2 * k + 1], o);
    for (int j = 0; j < 4; ++j) out[4 * k + j] = o[j];
}

// The variability prefilter on given inputs (profile pair rounded exactly as
// the host rounds it): out = var_prefilter code (bit 1: undecided, bit 0: +1).
__global__ void debug_var_prefilter(int64_t cnt, const double *lam, const double *delta,
                                    const double *i0, const int *raw, const uint32_t *zh,
                                    uint32_t *out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    const __half2 h = __floats2half2_rn((float)lam[k], (float)(lam[k] * delta[k]));
    const float ir = (float)i0[k] * (float)raw[k];
    out[k] = var_prefilter(h, ir, zh[k], 1.0f);
}

__global__ void debug_tanh(int64_t cnt, const double *x, double *out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < cnt) out[g] = pb_libm_tanh(x[g]);
}

}  // namespace pbsa
