// aux_kernels.cuh -- non-template kernels of the host runtime: spin init, first-absorb
// cache, general (int8) path, output formatting, debug hooks.  Included by the
// runtime units through runtime.h: the kernels have internal linkage (an
// unnamed namespace), each unit launching its own copy.
#pragma once
#include "device_common.cuh"

namespace pbsa {
namespace {

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
                                  int n, int chunks, int W, const uint32_t *__restrict__ order) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)W * chunks * 1024) return;
    const int lane = (int)(g & 31), b = (int)((g >> 5) & 31);
    const int64_t tile = g >> 10;
    const int ch = (int)(tile % chunks), w = (int)(tile / chunks);
    const int i = order ? (int)order[ch * 32 + lane] : ch * 32 + lane;  // (the sweep's node of this lane)
    uint64_t s = 0;
    if (i < n) s = mix64(krg[w * 32 + b] ^ (uint64_t)i) + PB_GAMMA;
    // store y' = s ^ (s >> 30): the sweep only XORs the sub-step counter into
    // its low word (count < 2^30 never reaches the shifted bits)
    const uint64_t y = s ^ (s >> 30);
    acache[tile * 1024 + cache_lane(lane) + cache_off(b)] = make_uint2((uint32_t)y, cache_hi_entry((uint32_t)(y >> 32)));
}


// Period buckets of the timing-spread sweep (packed_sweep_bucket): one warp
// per (word w, chunk ch) tile counting-sorts the tile's 1024 (lane, trial)
// slots by period class (lut: clamped period -> class, lanes past n get
// class nclass and are left out), trial-major inside a class so that a round
// of 32 consecutive slots touches many lanes' masks.  Each 16-byte record
// holds the slot, its fp16 (lam, lam delta) pair and the sub-step-independent
// first absorb of its replayed draw (as packed_cache_init: y' = s ^ (s >> 30),
// s = absorb(K_t, i) + GAMMA, stored as (low word, high word * M1L)); boff
// holds the class starts (boff[nclass] = the tile's record count).
__global__ void bucket_build(const uint32_t *__restrict__ pplanes, int nplanes,
                             const uint8_t *__restrict__ lut, const __half2 *__restrict__ prof16,
                             const uint64_t *__restrict__ krg, int n, int chunks, int W, int nclass,
                             uint4 *__restrict__ brec, uint16_t *__restrict__ boff,
                             const uint32_t *__restrict__ order) {
    __shared__ uint32_t cnt[8][257];
    __shared__ uint8_t slut[256];
    for (int k = threadIdx.x; k < 256; k += blockDim.x) slut[k] = lut[k];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    if (tile >= (int64_t)W * chunks) return;
    const int w = (int)(tile / chunks), ch = (int)(tile % chunks);
    const int i = order ? (int)order[ch * 32 + lane] : ch * 32 + lane;  // (the sweep's node of this lane)
    const bool valid = i < n;
    uint32_t pl[8];
    for (int k = 0; k < 8; ++k)
        pl[k] = (valid && k < nplanes) ? pplanes[((size_t)w * nplanes + k) * n + i] : 0u;
    uint32_t *c = cnt[wib];
    for (int k = lane; k <= nclass; k += 32) c[k] = 0;
    __syncwarp();
    int cls[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        int per = 0;
        for (int k = 0; k < nplanes; ++k) per |= (int)((pl[k] >> b) & 1u) << k;
        cls[b] = valid ? (int)slut[per] : nclass;
        atomicAdd(c + cls[b], 1u);
    }
    __syncwarp();
    uint4 *rec = brec + tile * 1024;
    // exclusive scan of the class counts -> class starts (cursors)
    uint32_t carry = 0;
    for (int k0 = 0; k0 <= nclass; k0 += 32) {
        const int k = k0 + lane;
        const uint32_t v = k < nclass ? c[k] : 0u;
        uint32_t incl = v;
        for (int sft = 1; sft < 32; sft <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, sft);
            if (lane >= sft) incl += t;
        }
        if (k <= nclass) {
            const uint32_t start = carry + incl - v;
            c[k] = start;
            boff[tile * (nclass + 1) + k] = (uint16_t)start;
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        const int k = cls[b];
        const uint32_t m = __match_any_sync(0xffffffffu, k);
        const uint32_t pos = c[k] + __popc(m & lt);
        __syncwarp();
        if ((m & lt) == 0) c[k] += __popc(m);
        __syncwarp();
        if (k < nclass) {
            const __half2 pv = prof16[((size_t)w * n + i) * 32 + b];
            uint32_t bits;
            memcpy(&bits, &pv, 4);
            const uint64_t s = mix64(krg[(size_t)w * 32 + b] ^ (uint64_t)i) + PB_GAMMA;
            const uint64_t y = s ^ (s >> 30);
            rec[pos] = make_uint4((uint32_t)((lane << 5) | b), bits, (uint32_t)y,
                                  (uint32_t)(y >> 32) * 0x1CE4E5B9u);
        }
    }
}

// Native variability profiles (rng = Philox, ExperimentSpec.native_profiles):
// the reference draws lam ~ N(1, s_l^2), delta ~ N(0, s_d^2) and the period
// max(1, rint(t_res (1 + nu))), nu ~ N(0, s_n^2), per p-bit with numpy
// (pbit.py:57-75); here the three normals of (global trial g, node i) come
// from one Philox4x32-10 block -- counter (i, g_hi, g_lo, tag 5) under the
// plan's native seed -- through two Box-Muller pairs (u = (X + 1/2) 2^-32),
// generated on the device at plan creation (no host sampling, no profile
// upload).  Padding trials get the ideal profile; periods are clamped to
// cycles * t_res, and a clamped period of 256 or more sets *overflow.
constexpr uint32_t kNativeTagProfile = 5u;

__device__ __forceinline__ void native_profile_of(uint32_t k0, uint32_t k1, uint64_t g, uint32_t i,
                                                  double sl, double sd, double sn, int t_res,
                                                  double &lam, double &del, int64_t &per) {
    uint32_t o[4];
    philox4x32_10(i, (uint32_t)(g >> 32), (uint32_t)g, kNativeTagProfile, k0, k1, o);
    const double u0 = ((double)o[0] + 0.5) * 0x1p-32, u1 = ((double)o[1] + 0.5) * 0x1p-32;
    const double u2 = ((double)o[2] + 0.5) * 0x1p-32, u3 = ((double)o[3] + 0.5) * 0x1p-32;
    const double r0 = sqrt(-2.0 * log(u0)), r1 = sqrt(-2.0 * log(u2));
    double s0, c0;
    sincospi(2.0 * u1, &s0, &c0);
    const double z3 = r1 * cospi(2.0 * u3);
    lam = 1.0 + sl * (r0 * c0);
    del = sd * (r0 * s0);
    const double nu = sn * z3;
    per = (int64_t)fmax(1.0, rint((double)t_res * (1.0 + nu)));
}

__global__ void native_profiles(uint32_t k0, uint32_t k1, uint64_t first_trial, int64_t T, int64_t Tp, int n,
                                int t_res, double sl, double sd, double sn, int64_t maxcount,
                                double *__restrict__ l64, double *__restrict__ d64,
                                uint8_t *__restrict__ pcl, int *__restrict__ overflow) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Tp * (int64_t)n) return;
    const int64_t t = g / n;
    const int i = (int)(g % n);
    if (t >= T) {
        l64[g] = 1.0;
        d64[g] = 0.0;
        return;
    }
    double lam, del;
    int64_t per;
    native_profile_of(k0, k1, first_trial + (uint64_t)t, (uint32_t)i, sl, sd, sn, t_res, lam, del, per);
    l64[g] = lam;
    d64[g] = del;
    const int64_t pc = per < maxcount ? per : maxcount;
    if (pc >= 256) atomicOr(overflow, 1);
    pcl[g] = (uint8_t)(pc < 256 ? pc : 255);
}

__global__ void fill_f64(double *__restrict__ p, int64_t n, double v) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) p[g] = v;
}

// The prefilter's profile pairs from the exact profile, rounded as the host
// rounds them: fp16 node-major [W][n][32] (timing spread) or fp32 [Tp][n].
__global__ void profile_pairs(const double *__restrict__ l64, const double *__restrict__ d64, int64_t Tp, int n,
                              __half2 *__restrict__ prof16, float2 *__restrict__ prof) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Tp * (int64_t)n) return;
    const int64_t t = g / n;
    const int i = (int)(g % n);
    const double lam = l64[g], ld = lam * d64[g];
    if (prof16)
        prof16[((size_t)(t >> 5) * n + i) * 32 + (t & 31)] = __floats2half2_rn((float)lam, (float)ld);
    else
        prof[g] = make_float2((float)lam, (float)ld);
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

}  // namespace
}  // namespace pbsa
