// device_common.cuh -- shared device helpers and kernel argument blocks of the
// B200-native pSA sweep (split from the round-1 monolith; see pbsa_device.cuh).
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
    const uint32_t *adj;      // [nnz] column | (J < 0) << 31 (n > 32768), else null
    const uint16_t *adj16;    // [nnz] column | (J < 0) << 15 (n <= 32768), else null
    const uint2 *kfc;         // [Tp] per-trial (F_t, C_t)
    const uint2 *acache;      // [W][chunks][32 trials][32 lanes] absorb(K_t, i) + GAMMA, or null
    const uint64_t *krg;      // [Tp] absorb(key, TAG_R) + GAMMA (exact slow path)
    const uint64_t *thr;      // [K] thresholds of this cycle (H >= thr -> +1)
    unsigned long long *pacc; // [Tp] += sum_i s_i * raw_i of the sub-step's input state
    int16_t *raw_out;         // [n][Tp] raw field of this update, or null
    int n, W, Tp, K, dmax;
    int warps_per_word;       // warps sharing one word index
    int cta_flush;            // every warp of a block has the same word: one cut flush per block
    int cache_prefetch;       // prefetch hash-cache tiles into L1 (phased plans: the cache is L2-resident)
    int grid2d;               // 2-D grid (warps_per_word / kPackedWarps, words): one word per block
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
    // BUCKET (timing spread, packed_sweep_bucket): each (word, 32-node chunk)
    // tile's 1024 (lane, trial) slots sorted by period class
    const uint4 *brec;        // [W][chunks][1024] class-sorted slot records: x = lane << 5 | trial
                              // bit, y = fp16 {lam, lam * delta} of that p-bit, (z, w) = its
                              // first-absorb cache (y' low word, y' high word * M1L)
    const uint16_t *boff;     // [W][chunks][nclass + 1] start of each class in the tile
    int nclass;               // distinct clamped periods present
    const uint8_t *cper;      // [nclass] clamped period of each class
    uint32_t maxcount;        // cycles * t_res
    const uint32_t *order;    // [chunks * 32] node processed by (chunk, lane) (degree order; n = none), or null
};

// Exact H >= thr for H = mix64(x); thr == ~0 encodes "never" (tanh == -1),
// which no genuine threshold equals (their low 11 bits are clear).
__device__ __forceinline__ bool hash_ge_exact(uint64_t x, uint64_t thr) {
    return mix64(x) >= thr && thr != ~0ULL;
}

#ifndef PBSA_PACKED_THREADS
#define PBSA_PACKED_THREADS 128
#endif
constexpr int kPackedThreads = PBSA_PACKED_THREADS;
constexpr int kPackedWarps = kPackedThreads / 32;
// packed_sweep's block-level cut reduction buffer: per warp up to 9 count
// planes and the degree sum, 32 lanes each
constexpr size_t kPackedFlushBytes = (size_t)kPackedWarps * 10 * 32 * 4 + 16;

__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }

// (lo, hi + add) of a 32 x 32 product.  WIDE: one IMAD.WIDE (+ the add)
// instead of a multiply and a multiply-high -- used by the plain sweep's
// decision only (C4 +1.5 %); in the period-bucket kernel it cost registers
// (G55 C3 +7 % time), elsewhere it compiled to the same code.
#ifndef PBSA_WIDE_MUL
#define PBSA_WIDE_MUL 1
#endif
template <bool WIDE = false>
__device__ __forceinline__ void mul_lohi(uint32_t a, uint32_t m, uint32_t add, uint32_t &lo, uint32_t &hi) {
    if (WIDE) {
        const uint64_t p = (uint64_t)a * m;
        lo = (uint32_t)p;
        hi = (uint32_t)(p >> 32) + add;
    } else {
        lo = a * m;
        hi = mulhi(a, m) + add;
    }
}

// First absorb of a trial's draw: s = absorb(K, i) + GAMMA, as (lo, hi).
// y = (ylo, Y) with ylo = F_t ^ i; Y * M1L is folded into C = C_t.
// Right shifts of high words go through IMAD.HI (x >> s == umulhi(x, 2^(32-s)))
// so the FMA pipe takes part of the load of the saturated ALU pipe.
__device__ __forceinline__ void packed_first_absorb(uint32_t ylo, uint32_t C, uint32_t &sl,
                                                    uint32_t &sh) {
    constexpr uint32_t M1L = 0x1CE4E5B9u, M1H = 0xBF58476Du;
    constexpr uint32_t M2L = 0x32684F87u, M2H = 0x94D4A04Cu;
    constexpr uint32_t GL = 0x7F4A7C15u, GH = 0x9E3779B9u;
    uint32_t zl, zh;
    mul_lohi(ylo, M1L, ylo * M1H + C, zl, zh);
    // z ^= z >> 27 ; z *= M2
    uint32_t yl = zl ^ __funnelshift_r(zl, zh, 27);
    uint32_t yh = zh ^ mulhi(zh, 1u << 5);
    mul_lohi(yl, M2L, yl * M2H + yh * M2L, zl, zh);
    // z ^= z >> 31  -> A ; s = A + GAMMA
    yl = zl ^ __funnelshift_r(zl, zh, 31);
    yh = zh ^ mulhi(zh, 1u << 1);
    asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
        : "=r"(sl), "=r"(sh) : "r"(yl), "r"(yh), "r"(GL), "r"(GH));
}

// Second absorb from y = x ^ (x >> 30), x = s ^ count, up to the high word of
// the last multiply, then the decision bit shifted into `word` through the
// carry of zh + ~thi.  Returns the (zh ^ thi) tie witness (< 2: recompute).
__device__ __forceinline__ uint32_t packed_decide_y(uint32_t yl, uint32_t c1, uint2 t,
                                                    uint32_t &word) {
    constexpr uint32_t M1L = 0x1CE4E5B9u, M1H = 0xBF58476Du;
    constexpr uint32_t M2L = 0x32684F87u, M2H = 0x94D4A04Cu;
    uint32_t zl, zh;
    mul_lohi(yl, M1L, yl * M1H + c1, zl, zh);
    yl = zl ^ __funnelshift_r(zl, zh, 27);
    const uint32_t yh = zh ^ mulhi(zh, 1u << 5);
    zh = mulhi(yl, M2L) + yl * M2H + yh * M2L;
    asm("{\n\t.reg .u32 lo;\n\tadd.cc.u32 lo, %1, %2;\n\taddc.u32 %0, %3, %3;\n\t}"
        : "=r"(word) : "r"(zh), "r"(t.x), "r"(word));
    return zh ^ t.y;
}

// High word zh of the last multiply of the second absorb, from its input
// y = x ^ (x >> 30) given as (low word, high word * M1L); the draw's top word
// is zh ^ (zh >> 31), within 1 of zh.
__device__ __forceinline__ uint32_t packed_hash_hi_c(uint32_t yl, uint32_t c1) {
    constexpr uint32_t M1L = 0x1CE4E5B9u, M1H = 0xBF58476Du;
    constexpr uint32_t M2L = 0x32684F87u, M2H = 0x94D4A04Cu;
    uint32_t zl, zh;
    mul_lohi(yl, M1L, yl * M1H + c1, zl, zh);
    yl = zl ^ __funnelshift_r(zl, zh, 27);
    const uint32_t yh = zh ^ mulhi(zh, 1u << 5);
    return mulhi(yl, M2L) + yl * M2H + yh * M2L;
}

// The hash cache entry of a (trial, node): (low word, high word x M1L) of
// y' = s ^ (s >> 30) with PBSA_CACHE_C1 (one multiply per update fewer), else
// (low word, high word); cache_c1 gives the c1 term either way.
#ifndef PBSA_CACHE_C1
#define PBSA_CACHE_C1 1
#endif
// Layout of a (word, 32-node chunk) tile of the hash cache (1024 entries of
// 8 B): with PBSA_CACHE_PAIRS trial pairs are interleaved per lane,
// [b / 2][lane][b % 2], so the plain sweep loads two trials with one 16-byte
// load, and every consumer loads pairs (cache_get); else [b][lane].
// cache_lane / cache_off give a lane's base and trial b's offset in entries.
#ifndef PBSA_CACHE_PAIRS
#define PBSA_CACHE_PAIRS 1
#endif
__host__ __device__ __forceinline__ int cache_lane(int lane) { return PBSA_CACHE_PAIRS ? 2 * lane : lane; }
__host__ __device__ __forceinline__ int cache_off(int b) { return PBSA_CACHE_PAIRS ? (b >> 1) * 64 + (b & 1) : b * 32; }
// Trial b's cache entry inside a loop over a lane's 32 trials.  With the pair
// layout the 16-byte load of (b & ~1, b | 1) happens at the first trial of the
// pair the loop visits (ASC: even b, else odd b) and `pr` carries it to the
// second; CS selects evict-first loads (the resident kernels), else the
// read-only path.
template <bool ASC, bool CS = false>
__device__ __forceinline__ uint2 cache_get(const uint2 *ctile, int b, uint4 &pr) {
    if (!PBSA_CACHE_PAIRS) return CS ? __ldcs(ctile + cache_off(b)) : __ldg(ctile + cache_off(b));
    if ((b & 1) == (ASC ? 0 : 1)) {
        const uint4 *q = reinterpret_cast<const uint4 *>(ctile + cache_off(b & ~1));
        pr = CS ? __ldcs(q) : __ldg(q);
    }
    return (b & 1) ? make_uint2(pr.z, pr.w) : make_uint2(pr.x, pr.y);
}

__device__ __forceinline__ uint32_t cache_c1(uint32_t hi) { return PBSA_CACHE_C1 ? hi : hi * 0x1CE4E5B9u; }
__host__ __device__ __forceinline__ uint32_t cache_hi_entry(uint32_t yh) {
    return PBSA_CACHE_C1 ? yh * 0x1CE4E5B9u : yh;
}

// Same from the first absorb s (x = s ^ count; count < 2^30 only touches the low word).
__device__ __forceinline__ uint32_t packed_hash_hi(uint32_t sl, uint32_t sh, uint32_t count) {
    return packed_hash_hi_c(sl ^ count ^ __funnelshift_r(sl, sh, 30), (sh ^ mulhi(sh, 1u << 2)) * 0x1CE4E5B9u);
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
    return packed_decide_y(sl ^ count ^ __funnelshift_r(sl, sh, 30), (sh ^ mulhi(sh, 1u << 2)) * 0x1CE4E5B9u,
                           t, word);
}

// Plain-rule variant with the table entry t = (lo, hi) of the 33-bit
// n2 = ~thi + 2: the carry of zh + n2 is zh >= thi - 1 and its low word is
// D = zh - thi + 1, so D < 3 (zh within 1 of thi, where the draw's low word
// or the final xorshift's bit 0 matter) is the only case that needs the
// exact 64-bit test, and every other carry is the exact decision -- also for
// thi <= 1, which the 33rd bit keeps.  Returns D.
__device__ __forceinline__ uint32_t packed_decide_n2(uint32_t yl, uint32_t c1, uint2 t,
                                                     uint32_t &word) {
    constexpr uint32_t M1L = 0x1CE4E5B9u, M1H = 0xBF58476Du;
    constexpr uint32_t M2L = 0x32684F87u, M2H = 0x94D4A04Cu;
    uint32_t zl, zh;
    mul_lohi<PBSA_WIDE_MUL != 0>(yl, M1L, yl * M1H + c1, zl, zh);
    yl = zl ^ __funnelshift_r(zl, zh, 27);
    const uint32_t yh = zh ^ mulhi(zh, 1u << 5);
    zh = mulhi(yl, M2L) + yl * M2H + yh * M2L;
    uint32_t D;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
        : "=r"(D), "=r"(word) : "r"(zh), "r"(t.x), "r"(word), "r"(word + t.y));
    return D;
}

__device__ __forceinline__ uint32_t packed_second_decide_n2(uint32_t sl, uint32_t sh, uint32_t count,
                                                            uint2 t, uint32_t &word) {
    return packed_decide_n2(sl ^ count ^ __funnelshift_r(sl, sh, 30), (sh ^ mulhi(sh, 1u << 2)) * 0x1CE4E5B9u,
                            t, word);
}

// Native decision: shift (X >= T) into `word` as the carry of X + (2^32 - T),
// t = (lo, hi) of the 33-bit 2^32 - T (T = 2^32 never fires, T = 0 always).
__device__ __forceinline__ void native_decide(uint32_t X, uint2 t, uint32_t &word) {
    asm("{\n\t.reg .u32 lo;\n\tadd.cc.u32 lo, %1, %2;\n\taddc.u32 %0, %3, %4;\n\t}"
        : "=r"(word) : "r"(X), "r"(t.x), "r"(word), "r"(word + t.y));
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

// blocks per SM of the period-bucket kernel: 8 (64 registers) for the tori
// (L <= 3), 6 (85 registers) otherwise; measured with 256 staged records:
// G81 C3 -5.6 % against 6 blocks, G55 C3 +0 / -19 % with 7 / 8 blocks
#ifndef PBSA_BUCKET_MIN_BLOCKS
#define PBSA_BUCKET_MIN_BLOCKS 6
#endif
#ifndef PBSA_BUCKET_MIN_BLOCKS_L3
#define PBSA_BUCKET_MIN_BLOCKS_L3 8
#endif
#ifndef PBSA_PACKED_MIN_BLOCKS
#define PBSA_PACKED_MIN_BLOCKS 8
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
#ifndef PBSA_MASKED_TAIL
#define PBSA_MASKED_TAIL 1
#endif
template <int L, bool MASKED = true, typename NB>
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
    // (called for L >= 3 only; the clamped plane indices keep the L < 3
    // instances well-formed)
    constexpr int P1 = L > 1 ? 1 : 0, P2 = L > 2 ? 2 : 0;
    auto batch8 = [&](const uint32_t (&x)[8]) {
        uint32_t twosA, twosB, foursA, foursB, eights;
        csa(twosA, p[0], x[0], x[1]);
        csa(twosB, p[0], x[2], x[3]);
        csa(foursA, p[P1], twosA, twosB);
        csa(twosA, p[0], x[4], x[5]);
        csa(twosB, p[0], x[6], x[7]);
        csa(foursB, p[P1], twosA, twosB);
        csa(eights, p[P2], foursA, foursB);
        ripple(eights, 3);
    };
    if (L >= 4) {
        for (; k + 8 <= end; k += 8) {
            uint32_t x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = nb(k + j);
            batch8(x);
        }
    }
    if (L >= 3 && MASKED && PBSA_MASKED_TAIL) {
        // the remaining (< 8) entries as one masked batch, their loads in flight
        // together instead of one dependent load pair per entry; absent entries
        // add zero (and a sum below 2^L leaves the weight-8 digit zero for L = 3)
        if (k < end) {
            uint32_t x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = k + j < end ? nb(k + j) : 0u;
            batch8(x);
        }
    } else {
        for (; k < end; ++k) ripple(nb(k), 0);
    }
}

template <int L, bool MASKED = true>
__device__ __forceinline__ void gather_counts(const uint32_t *__restrict__ adj,
                                              const uint32_t *__restrict__ sw, uint32_t beg,
                                              uint32_t end, uint32_t (&p)[L]) {
    count_neighbours<L, MASKED>(beg, end, [&](uint32_t k) {
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

// The device CSR (model.py:21-33 row order): 16-bit entries column | (J < 0)
// << 15 whenever n <= 32768 (every G-set graph: G81's 80k couplings in 160 KB,
// so a CTA's slice, or the whole graph, sits in shared memory), 32-bit column
// | (J < 0) << 31 beyond.  Kernels branch once per node on which is present.
__device__ __forceinline__ uint32_t adj16_to32(uint32_t e16) {
    return (e16 & 0x7fffu) | ((e16 & 0x8000u) << 16);
}

// Node handled by lane `lane` of 32-node chunk `ch`: the identity, or, on
// irregular graphs, a degree-sorted processing order (nodes of similar degree
// share a warp, so its gather loop runs ~ their degree instead of the maximum
// of 32 random degrees).  Labels, spin layout and draws are unchanged.
template <typename A>
__device__ __forceinline__ int node_at(const A &a, int ch, int lane) {
    const int k = ch * 32 + lane;
    return a.order ? (int)__ldg(a.order + k) : k;
}

template <int L, bool MASKED = true>
__device__ __forceinline__ void gather_counts16(const uint16_t *__restrict__ adj,
                                                const uint32_t *__restrict__ sw, uint32_t beg,
                                                uint32_t end, uint32_t (&p)[L]) {
    count_neighbours<L, MASKED>(beg, end, [&](uint32_t k) {
        const uint32_t e = __ldg(adj + k);
        return __ldg(sw + (e & 0x7fffu)) ^ (0u - (e >> 15));
    }, p);
}

template <int L, bool MASKED = true, typename A>
__device__ __forceinline__ void gather_rows(const A &a, const uint32_t *__restrict__ sw, uint32_t beg,
                                            uint32_t end, uint32_t (&p)[L]) {
    if (a.adj16)
        gather_counts16<L, MASKED>(a.adj16, sw, beg, end, p);
    else
        gather_counts<L, MASKED>(a.adj, sw, beg, end, p);
}

// Degree-4 rows: the raw row of node i (16-bit: its four entries in .x, .y)
// and its 32-bit form for gather_counts_row4.
template <typename A>
__device__ __forceinline__ uint4 load_row4(const A &a, int i) {
    if (a.adj16) {
        const uint2 u = __ldg(reinterpret_cast<const uint2 *>(a.adj16) + i);
        return make_uint4(u.x, u.y, 0u, 0u);
    }
    return __ldg(reinterpret_cast<const uint4 *>(a.adj) + i);
}

// 16-bit degree-4 row (entries e.x lo/hi, e.y lo/hi): as gather_counts_row4
// bit-sliced x0 + x1 + x2 + x3 (<= 4 < 2^L, L >= 3 since dmax = 4)
template <int L>
__device__ __forceinline__ void add4_planes(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t (&p)[L]) {
    const uint32_t s01 = x0 ^ x1, c01 = x0 & x1, s23 = x2 ^ x3, c23 = x2 & x3;
    const uint32_t s = s01 ^ s23, cs = s01 & s23;
    const uint32_t t = c01 ^ c23 ^ cs;
    const uint32_t f = (c01 & c23) | (cs & (c01 ^ c23));
#pragma unroll
    for (int r = 0; r < L; ++r) p[r] = r == 0 ? s : r == 1 ? t : r == 2 ? f : 0u;
}

template <int L>
__device__ __forceinline__ void gather_counts_row4_16(const uint4 e, const uint32_t *__restrict__ sw,
                                                      uint32_t (&p)[L]) {
    const uint32_t x0 = __ldg(sw + (e.x & 0x7fffu)) ^ (0u - ((e.x >> 15) & 1u));
    const uint32_t x1 = __ldg(sw + ((e.x >> 16) & 0x7fffu)) ^ (uint32_t)((int32_t)e.x >> 31);
    const uint32_t x2 = __ldg(sw + (e.y & 0x7fffu)) ^ (0u - ((e.y >> 15) & 1u));
    const uint32_t x3 = __ldg(sw + ((e.y >> 16) & 0x7fffu)) ^ (uint32_t)((int32_t)e.y >> 31);
    const uint32_t s01 = x0 ^ x1, c01 = x0 & x1, s23 = x2 ^ x3, c23 = x2 & x3;
    const uint32_t s = s01 ^ s23, cs = s01 & s23;
    const uint32_t t = c01 ^ c23 ^ cs;
    const uint32_t f = (c01 & c23) | (cs & (c01 ^ c23));
#pragma unroll
    for (int r = 0; r < L; ++r) p[r] = r == 0 ? s : r == 1 ? t : r == 2 ? f : 0u;
}

template <int L, typename A>
__device__ __forceinline__ void gather_row4(const A &a, const uint4 e, const uint32_t *__restrict__ sw,
                                            uint32_t (&p)[L]) {
    if (a.adj16)
        gather_counts_row4_16<L>(e, sw, p);
    else
        gather_counts_row4<L>(e, sw, p);
}

template <typename A>
__device__ __forceinline__ uint4 expand_row4(const A &a, uint4 e) {
    if (!a.adj16) return e;
    return make_uint4(adj16_to32(e.x & 0xffffu), adj16_to32(e.x >> 16), adj16_to32(e.y & 0xffffu),
                      adj16_to32(e.y >> 16));
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

constexpr int kMaxDivisors = 256;
// packed_sweep_bucket shared memory: per-warp keys; per warp a staging list
// of the tile's fired slot records (16 bytes each, bulk-copied, kBucketStage
// records), its mbarrier, scratch (count planes, own word, degree, flip and
// exact masks: u32 per lane) and the u16 segment table (prefix, start per
// fired class); the launch's class list and last-firing flags.
#ifndef PBSA_BK_STAGE
#define PBSA_BK_STAGE 256  // (384: G81 C3 +5.6 %, G55 C3 +10 % time)
#endif
constexpr int kBucketStage = PBSA_BK_STAGE;            // staged records per tile (the rest load directly)
constexpr int kBucketMaxDiv = 128;            // fired classes per sub-step the bucket kernel takes
constexpr int kBucketSegs = kBucketMaxDiv + 1;
__host__ __device__ constexpr int bucket_scratch(int L) { return ((L < 4 ? 4 : L) + 5) * 32; }
__host__ __device__ constexpr size_t bucket_warp_bytes(int L) {
    return (kBucketStage * 16 + 16 + bucket_scratch(L) * 4 + 2 * kBucketSegs * 2 + 15) / 16 * 16;
}
__host__ __device__ constexpr size_t bucket_smem_bytes(int L) {
    return kPackedWarps * 32 * 8 + kPackedWarps * bucket_warp_bytes(L) + kBucketMaxDiv * 3;
}
constexpr size_t kTimingSmem = kPackedWarps * 32 * sizeof(uint2) + kMaxDivisors * 8 * 4 +
                               2 * kPackedWarps * 32 * 4 + kPackedWarps * 1024 * 4;


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
    const uint16_t *adj16;      // [nnz] column | (J < 0) << 15 (resident plans have n <= 32768)
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
    const uint32_t *rowptr;
    const uint16_t *adj16;      // [nnz] column | (J < 0) << 15
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

}  // namespace pbsa
