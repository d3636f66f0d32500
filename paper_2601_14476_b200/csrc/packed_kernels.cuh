// packed_kernels.cuh -- launched packed sweeps (one launch per sub-step): packed_sweep
// (plain / TApSA / SpSA / varied profile, replayed or Philox draws) and the
// timing-spread sweep.  Instantiated per degree width L in kernels_L*.cu.
#pragma once
#include <type_traits>

#include "device_common.cuh"

namespace pbsa {

// hash-cache loads: 0 evict-first (ld.global.cs), 1 read-only path (ld.global.nc;
// measured +1 % over 0 once the tiles are prefetched into L1),
// 2 default caching
#ifndef PBSA_CACHE_LD
#define PBSA_CACHE_LD 1
#endif
__device__ __forceinline__ uint2 cache_ld(const uint2 *p) {
    if (PBSA_CACHE_LD == 1) return __ldg(p);
    if (PBSA_CACHE_LD == 2) return *p;
    return __ldcs(p);
}
__device__ __forceinline__ uint4 cache_ld2(const uint2 *p) {  // trials b - 1, b (b odd)
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
    if (PBSA_CACHE_LD == 1) return __ldg(q);
    if (PBSA_CACHE_LD == 2) return *q;
    return __ldcs(q);
}
// A warp's word w (within the launch) and its slot q among the word's
// warps_per_word warps.  With one word per block the grid may be 2-D,
// (warps_per_word / kPackedWarps, words), and no division is needed.
__device__ __forceinline__ void word_and_slot(const PackedArgs &a, int wib, int &w, int &q) {
    if (a.grid2d) {
        w = (int)blockIdx.y;
        q = (int)blockIdx.x * kPackedWarps + wib;
    } else {
        const int g = (int)blockIdx.x * kPackedWarps + wib;
        w = g / a.warps_per_word;
        q = g % a.warps_per_word;
    }
}
// PBSA_CACHE_PREFETCH: 1 prefetches a warp's first hash-cache tile into L1
// ahead of the dependent-launch wait, 2 also each next tile; 0 none.  At run
// time off by default (a.cache_prefetch: it measured +4 % on C4 mid-round 2
// and -2.3 % after the instruction trims)
#ifndef PBSA_CACHE_PREFETCH
#define PBSA_CACHE_PREFETCH 2
#endif
#ifndef PBSA_PRMT_ADDR
#define PBSA_PRMT_ADDR 1
#endif
// Blocks per SM the plain cached sweep is compiled for, per count width
// (registers = 64K / (128 x blocks)): measured per instance, since more
// registers let the compiler keep more of a chunk's 32 hash-cache loads in
// flight while fewer cost warps (A/B on one B200: see DESIGN.md section 4).
#ifndef PBSA_MB_L3
#define PBSA_MB_L3 7
#endif
#ifndef PBSA_MB_L4
#define PBSA_MB_L4 8
#endif
#ifndef PBSA_MB_L5
#define PBSA_MB_L5 PBSA_PACKED_MIN_BLOCKS
#endif
#ifndef PBSA_MB_L6
#define PBSA_MB_L6 PBSA_PACKED_MIN_BLOCKS
#endif
#ifndef PBSA_MB_L7
#define PBSA_MB_L7 6
#endif
// The Philox plain (ALG 4) and varied-profile (5) update sweeps spill at 64
// registers: 72 for L = 3 (G81 C4 Philox +1 %), 80 otherwise (G55 x 4096 +12 %,
// G1 x 4096 +27 %, G81 sigma_lam,delta +5 %).  TApSA / SpSA / replayed
// varied-profile sweeps lose with fewer blocks (G81 TApSA -11 %): 64.
#ifndef PBSA_MB_PHILOX_L3
#define PBSA_MB_PHILOX_L3 7
#endif
#ifndef PBSA_MB_PHILOX
#define PBSA_MB_PHILOX 6
#endif
#ifndef PBSA_MB_TAPSA
#define PBSA_MB_TAPSA 7  // (TApSA G81 / G55 x 4096 -3 / -5 % time against 8)
#endif
template <int L, bool UPDATE, bool CACHED, int ALG>
constexpr int packed_min_blocks() {
    return (UPDATE && CACHED && ALG == 0)
               ? (L == 3 ? PBSA_MB_L3 : L == 4 ? PBSA_MB_L4 : L == 5 ? PBSA_MB_L5 : L == 6 ? PBSA_MB_L6
                  : L == 7 ? PBSA_MB_L7 : PBSA_PACKED_MIN_BLOCKS)
           : (UPDATE && ALG == 4) ? (L == 3 ? PBSA_MB_PHILOX_L3 : PBSA_MB_PHILOX)
           : (UPDATE && ALG == 5) ? PBSA_MB_PHILOX
           : (UPDATE && ALG == 1) ? PBSA_MB_TAPSA
                                  : PBSA_PACKED_MIN_BLOCKS;
}

template <int L, bool UPDATE, bool CACHED, int ALG = 0>
__global__ void __launch_bounds__(kPackedThreads, (packed_min_blocks<L, UPDATE, CACHED, ALG>())) packed_sweep(PackedArgs a) {
    asm volatile("griddepcontrol.launch_dependents;");
    // (declared 1 KB-aligned: the table base is then a known shared-window
    // address, so its accesses compile to STS / LDS rather than generic ones)
    extern __shared__ __align__(1024) unsigned long long smem_pk[];
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
    // NIB rows: one per degree, kNibRow entries of 8 B (256 B with PBSA_PRMT_ADDR,
    // so a row base has a zero low byte and one PRMT forms a trial's address)
    constexpr int kNibRow = PBSA_PRMT_ADDR ? 32 : 16;
    uint2 *sthr = reinterpret_cast<uint2 *>(smem_pk);
    const int tab_entries = VAR ? 0 : TAPSA ? a.K : NIB ? (a.dmax + 1) * kNibRow : a.K;
    uint2 *skey = sthr + tab_entries;                     // [warps][32] {F, C}

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int w, q;
    word_and_slot(a, wib, w, q);
    const bool live = w < a.W;

    for (int k = threadIdx.x; k < tab_entries; k += blockDim.x) {
        uint32_t thi;
        uint64_t tfull = 0;  // NATIVE: the 33-bit Philox threshold T
        if (TAPSA) {
            tfull = a.thr[k];  // host table is already [acc + f dmax]
            thi = (uint32_t)(tfull >> 32);
        } else {
            int raw = k - a.dmax;
            if (NIB) {
                const int d = k / kNibRow, pp = k % kNibRow;
                if (pp > d) continue;  // (a count never exceeds the degree: never read)
                raw = 2 * pp - d;
            }
            tfull = a.thr[raw + a.dmax];
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
    // the first chunk's 8 KB hash-cache tile into L1 before waiting on the
    // previous sub-step (it does not depend on the spins): 64 lines, two per lane
    if (CACHED && PBSA_CACHE_PREFETCH && a.cache_prefetch && live && q < a.chunks) {
        const char *tile = reinterpret_cast<const char *>(a.acache + ((size_t)w * a.chunks + q) * 1024);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(tile + lane * 128));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(tile + 4096 + lane * 128));
    }
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
        uint4 e_nx = make_uint4(0u, 0u, 0u, 0u);
        uint32_t own_nx = 0;
        if (R4 && q < a.chunks && q * 32 + lane < a.n) {
            e_nx = load_row4(a, q * 32 + lane);
            own_nx = __ldg(sw + q * 32 + lane);
        }
        for (int ch = q; ch < a.chunks; ch += a.warps_per_word) {
            if (CACHED && PBSA_CACHE_PREFETCH > 1 && a.cache_prefetch && ch + a.warps_per_word < a.chunks) {
                const char *tile = reinterpret_cast<const char *>(
                    a.acache + ((size_t)w * a.chunks + ch + a.warps_per_word) * 1024);
                asm volatile("prefetch.global.L1 [%0];" ::"l"(tile + lane * 128));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(tile + 4096 + lane * 128));
            }
            const int i = node_at(a, ch, lane);
            if (i >= a.n) continue;
            uint32_t p[L];
            int d;
            uint32_t own;
            if (R4) {
                const uint4 e = e_nx;
                own = own_nx;
                const int ni = i + 32 * a.warps_per_word;
                if (ni < a.n) {
                    e_nx = load_row4(a, ni);
                    own_nx = __ldg(sw + ni);
                }
                gather_row4<L>(a, e, sw, p);
                d = 4;
            } else {
                const uint32_t beg = __ldg(a.rowptr + i), end = __ldg(a.rowptr + i + 1);
                own = __ldg(sw + i);
                gather_rows<L>(a, sw, beg, end, p);
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
                const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + ch) * 1024 + cache_lane(lane) : nullptr;
                uint32_t word = 0, exact = 0;
                uint32_t X[4];  // NATIVE: the current Philox block (trials 4k .. 4k + 3)
                uint4 cpair = make_uint4(0u, 0u, 0u, 0u);  // CACHED: the current trial pair
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
                        const uint2 v = cache_get<true>(ctile, b, cpair);
                        zh = packed_hash_hi_c(v.x ^ count, cache_c1(v.y));
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
                const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + ch) * 1024 + cache_lane(lane) : nullptr;
                uint32_t word = 0, tie = 0xffffffffu;
                const uint32_t ui = (uint32_t)i;
                uint32_t X[4];  // NATIVE: the current Philox block
                uint4 cpair = make_uint4(0u, 0u, 0u, 0u);  // CACHED: the current trial pair
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
                        const uint2 v = cache_get<false>(ctile, b, cpair);
                        tie = min(tie, packed_decide_y(v.x ^ count, cache_c1(v.y), t, word));
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
                const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + ch) * 1024 + cache_lane(lane) : nullptr;
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
                uint4 cpair = make_uint4(0u, 0u, 0u, 0u);  // CACHED: the current trial pair
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
                            t = NIB ? sthr[d * kNibRow + pop] : sthr[2 * pop - d + a.dmax];
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
                            const uint2 v = cache_get<false>(ctile, b, cpair);
                            tie = min(tie, packed_decide_y(v.x ^ count, cache_c1(v.y), t, word));
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
                const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + ch) * 1024 + cache_lane(lane) : nullptr;
                uint32_t word = 0, tie = 0xffffffffu;
                const uint32_t ui = (uint32_t)i;
                uint32_t X[4];  // NATIVE: the current Philox block (trials 4k .. 4k + 3)
                uint4 cpair = make_uint4(0u, 0u, 0u, 0u);  // CACHED: the current trial pair
                // NIB: transpose the L count planes into 32 nibbles (N[k] nibble j =
                // count of trial 8k + j), a few ops per 32 trials instead of 2L per trial;
                // PBSA_PRMT_ADDR: into bytes holding 8 x count (B[k] byte j = trial
                // 4k + j; four trials' bits spread by one multiply), so that a trial's
                // table address is one PRMT of its byte with the row base
                uint32_t N[4] = {0u, 0u, 0u, 0u};
                uint32_t B8[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                uint32_t rb = 0;
                if (NIB && PBSA_PRMT_ADDR) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
#pragma unroll
                        for (int r = 0; r < L; ++r) {
                            const uint32_t x4 = (p[r] >> (4 * k)) & 0xFu;
                            B8[k] |= (x4 * (0x00204081u << (r + 3))) & (0x01010101u << (r + 3));
                        }
                    }
                    rb = (uint32_t)__cvta_generic_to_shared(sthr) + (uint32_t)d * (8u * kNibRow);
                } else if (NIB) {
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
                    if (NIB && PBSA_PRMT_ADDR) {
                        const uint32_t addr = __byte_perm(B8[b >> 2], rb, 0x7650u | (uint32_t)(b & 3));
                        asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(t.x), "=r"(t.y) : "r"(addr));
                    } else if (NIB) {
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
                        native_decide(X[b & 3], t, word);
                    } else if (CACHED) {
                        const uint2 v = cache_get<false>(ctile, b, cpair);
                        tie = min(tie, packed_decide_n2(v.x ^ count, cache_c1(v.y), t, word));
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
    if (a.cta_flush) {
        // every warp of the block works on word w (warps_per_word is a multiple
        // of the block's warps): add the warps' bit-sliced counters in shared
        // memory and flush once per block instead of once per warp
        uint32_t *sC = scount + 4;                                   // [warps][CP][32]
        int *sD = reinterpret_cast<int *>(sC + kPackedWarps * CP * 32);  // [warps][32]
#pragma unroll
        for (int r = 0; r < CP; ++r) sC[(wib * CP + r) * 32 + lane] = C[r];
        sD[wib * 32 + lane] = dsum;
        __syncthreads();
        if (wib == 0) {
            constexpr int CQ = CP + 3;  // sums of up to 8 warps
            uint32_t S[CQ];
#pragma unroll
            for (int r = 0; r < CQ; ++r) S[r] = r < CP ? C[r] : 0u;
            for (int v = 1; v < kPackedWarps; ++v) {
                uint32_t x[CP];
#pragma unroll
                for (int r = 0; r < CP; ++r) x[r] = sC[(v * CP + r) * 32 + lane];
                vc_add<CP, CQ>(S, x);
                dsum += sD[v * 32 + lane];
            }
            warp_cut_flush(S, dsum, lane, live ? a.pacc + (size_t)w * 32 : nullptr);
        }
        return;
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
    int w, q;
    word_and_slot(a, wib, w, q);
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
            const int i = node_at(a, ch, lane);
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
                    gather_row4<L>(a, load_row4(a, i), sw, p);
                    d = 4;
                } else {
#pragma unroll
                    for (int r = 0; r < L; ++r) p[r] = 0;
                }
            } else {
                gather_rows<L>(a, sw, beg, end, p);
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
                const int ii = node_at(a, ch, l);
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
                return __ldg(a.prof16 + ((size_t)w * a.n + node_at(a, ch, (int)((e >> 5) & 31u))) * 32 + (e & 31u));
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
    if (a.do_cut)  // (the cut is taken on a cycle's first sub-step only)
        warp_cut_flush(C, dsum, lane, live ? a.pacc + (size_t)w * 32 : nullptr);
}

// ------------------------------------------- packed sweep over period buckets
// The timing-spread sweep without re-reading the variability profile of the
// p-bits that do not fire.  At plan creation every (word w, 32-node chunk ch)
// tile's 1024 (lane, trial) slots are counting-sorted by period class
// (bucket_build): `brec` lists the slots class by class, each with its fp16
// (lam, lam delta) pair and its draw's first-absorb cache, and `boff` holds
// the start of each class.  In
// sub-step `count` exactly the classes whose period divides it fire
// (_kernels.py:126), so a warp reads only those segments -- coalesced, about
// E[1/period] of the profile per sub-step -- instead of every fired p-bit's
// scattered pair plus the bit-sliced periods (packed_sweep_timing).
//
// Per tile the fired segments are bulk-copied (cp.async.bulk, one copy per
// class issued by that class's lane, completion on a per-warp mbarrier) into a
// shared-memory staging list while the warp gathers; the next tile's class
// bounds are loaded a tile ahead.  The gather forms the bit-sliced counts p[L]
// of the lane's node and parks them (with own word and degree) in shared
// memory; the warp deals the staged slots round-robin to its lanes, four per
// lane and round: slot (l, b) reads trial b's count from lane l's planes,
// draws, and decides with the variability prefilter; a decision that differs
// from the current spin sets the slot's bit in a flip mask, an undecided one
// its bit in the exact-recheck mask (shared memory).  The owner lane then
// writes own ^ flips, the exact fp64 recheck (_kernels.py:150-152) filling in
// the undecided trials.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// (PBSA_BK_NIB=1: counts as nibble tables; measured 3-5 % slower, kept off)
#ifndef PBSA_BK_NIB
#define PBSA_BK_NIB 0
#endif
#ifndef PBSA_BK_ILP
#define PBSA_BK_ILP 1
#endif
#ifndef PBSA_BK_NB_EARLY
#define PBSA_BK_NB_EARLY 1
#endif
template <int L, bool NATIVE = false>
__global__ void __launch_bounds__(kPackedThreads, L <= 3 ? PBSA_BUCKET_MIN_BLOCKS_L3 : PBSA_BUCKET_MIN_BLOCKS)
    packed_sweep_bucket(PackedArgs a) {
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ unsigned long long smem_u64[];
    constexpr size_t WB = bucket_warp_bytes(L);
    uint2 *skey = reinterpret_cast<uint2 *>(smem_u64);                      // [warps][32]
    uint8_t *swarp = reinterpret_cast<uint8_t *>(skey + kPackedWarps * 32);  // [warps][WB]
    uint16_t *sdiv = reinterpret_cast<uint16_t *>(swarp + kPackedWarps * WB);  // [kBucketMaxDiv]
    uint8_t *slast = reinterpret_cast<uint8_t *>(sdiv + kBucketMaxDiv);       // [kBucketMaxDiv]
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int w, q;
    word_and_slot(a, wib, w, q);
    const bool live = w < a.W;
    uint2 *key = skey + wib * 32;
    key[lane] = live ? a.kfc[(size_t)w * 32 + lane] : make_uint2(0, 0);
    uint8_t *wbase = swarp + wib * WB;
    uint4 *stage = reinterpret_cast<uint4 *>(wbase);                           // [kBucketStage]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(stage + kBucketStage);
    uint32_t *splane = reinterpret_cast<uint32_t *>(mbar + 2);                 // [max(L, 4)][32]
    uint32_t *sown = splane + (L < 4 ? 4 : L) * 32, *sdeg = sown + 32, *sflip = sdeg + 32, *sexm = sflip + 32;
    uint32_t *snode = sexm + 32;  // node of each lane of the tile
    uint16_t *pre = reinterpret_cast<uint16_t *>(snode + 32), *beg16 = pre + kBucketSegs;
    if (lane == 0) mbar_init(mbar, 1);
    // fired classes of this sub-step; a class whose period p has count + p >=
    // cycles * t_res fires here for the last time, so only its slots record
    // the input (i0 * raw of the last firing, _kernels.py:146)
    for (int k = threadIdx.x; k < a.ndiv; k += blockDim.x) {
        const uint32_t c = a.divs[k];
        sdiv[k] = (uint16_t)c;
        slast[k] = a.inp_out && a.count + a.cper[c] >= a.maxcount ? 1 : 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t count = a.count;
    constexpr int CP = CutPlanes<L>::value;
    uint32_t C[CP];
#pragma unroll
    for (int r = 0; r < CP; ++r) C[r] = 0;
    int dsum = 0;

    if (live) {
        const uint32_t *sw = a.sold + (size_t)w * a.n;
        const bool reg4 = L >= 3 && a.reg4;
        const size_t ncl1 = (size_t)a.nclass + 1;
        // class bounds (begin, end) of the lane's fired class k0 + lane in tile ch.
        // The next tile's are loaded a tile ahead; on the tori (L <= 3) they stay
        // the two loaded values until used (combining them at once waited on the
        // loads: G81 C3 +1 %), otherwise packed beg | end << 16 (one register
        // fewer: the L = 4 kernel keeps 7 blocks per SM, G55 C3 +6 %)
        using Bounds = std::conditional_t<(L <= 3), uint2, uint32_t>;
        auto bounds = [&](int ch, int k0) -> Bounds {
            const int k = k0 + lane;
            if (ch >= a.chunks || k >= a.ndiv) return Bounds{};
            const uint16_t *row = a.boff + ((size_t)w * a.chunks + ch) * ncl1 + sdiv[k];
            if constexpr (L <= 3)
                return make_uint2((uint32_t)__ldg(row), (uint32_t)__ldg(row + 1));
            else
                return (uint32_t)__ldg(row) | ((uint32_t)__ldg(row + 1) << 16);
        };
        auto bounds_beg_end = [](Bounds v, int &beg, int &end) {
            if constexpr (L <= 3) {
                beg = (int)v.x;
                end = (int)v.y;
            } else {
                beg = (int)(v & 0xFFFFu);
                end = (int)(v >> 16);
            }
        };
        Bounds bb_nx = bounds(q, 0);
        uint4 e_nx = make_uint4(0u, 0u, 0u, 0u);
        uint32_t own_nx = 0;
        if (reg4 && q < a.chunks && q * 32 + lane < a.n) {
            e_nx = load_row4(a, q * 32 + lane);
            own_nx = __ldg(sw + q * 32 + lane);
        }
        uint32_t parity = 0;
        for (int ch = q; ch < a.chunks; ch += a.warps_per_word, parity ^= 1u) {
            const int i = node_at(a, ch, lane);
            const bool valid = i < a.n;
            const uint4 *src = a.brec + ((size_t)w * a.chunks + ch) * 1024;
            // degree-4 16-bit rows: the tile's four neighbour words are loaded
            // before the segment scan, which then runs while they are in flight
            uint32_t xr[4] = {0u, 0u, 0u, 0u};
            const bool early_nb = PBSA_BK_NB_EARLY && L <= 3 && reg4 && a.adj16 && valid;  // (L > 3: registers)
            if (early_nb) {
                xr[0] = __ldg(sw + (e_nx.x & 0x7fffu));
                xr[1] = __ldg(sw + ((e_nx.x >> 16) & 0x7fffu));
                xr[2] = __ldg(sw + (e_nx.y & 0x7fffu));
                xr[3] = __ldg(sw + ((e_nx.y >> 16) & 0x7fffu));
            }
            // 1. the tile's fired segments (sizes even): prefix sums, and the
            // first kBucketStage records bulk-copied into the staging list
            int F = 0;
            uint32_t staged = 0;  // bytes in flight
            for (int k0 = 0; k0 < a.ndiv; k0 += 32) {
                const Bounds bb = k0 == 0 ? bb_nx : bounds(ch, k0);
                int beg, bend;
                bounds_beg_end(bb, beg, bend);
                const int sz = bend - beg;
                int incl = sz;
#pragma unroll
                for (int sft = 1; sft < 32; sft <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, sft);
                    if (lane >= sft) incl += v;
                }
                const int excl = F + incl - sz;
                const int nst = max(0, min(sz, kBucketStage - excl));  // this class's staged records
                if (k0 + lane < a.ndiv) {
                    pre[k0 + lane] = (uint16_t)excl;
                    beg16[k0 + lane] = (uint16_t)beg;
                    if (nst > 0) bulk_copy_g2s(stage + excl, src + beg, 16u * (uint32_t)nst, mbar);
                }
                staged += 16u * (uint32_t)__reduce_add_sync(0xffffffffu, (uint32_t)nst);
                F += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) {
                pre[a.ndiv] = (uint16_t)F;
                mbar_arrive_expect_tx(mbar, staged);
            }
            const int chn = ch + a.warps_per_word;
            bb_nx = bounds(chn, 0);
            // 2. gather: bit-sliced counts of the lane's node
            uint32_t own = 0;
            uint32_t p[L];
            int d = 0;
            if (reg4) {
                const uint4 er = e_nx;
                own = own_nx;
                const int ni = i + 32 * a.warps_per_word;
                if (ni < a.n) {
                    e_nx = load_row4(a, ni);
                    own_nx = __ldg(sw + ni);
                }
                if (early_nb) {
                    add4_planes<L>(xr[0] ^ (0u - ((er.x >> 15) & 1u)), xr[1] ^ (uint32_t)((int32_t)er.x >> 31),
                                   xr[2] ^ (0u - ((er.y >> 15) & 1u)), xr[3] ^ (uint32_t)((int32_t)er.y >> 31), p);
                    d = 4;
                } else if (valid) {
                    gather_row4<L>(a, er, sw, p);
                    d = 4;
                } else {
#pragma unroll
                    for (int r = 0; r < L; ++r) p[r] = 0;
                }
            } else {
                uint32_t beg = 0, end = 0;
                if (valid) {
                    beg = __ldg(a.rowptr + i);
                    end = __ldg(a.rowptr + i + 1);
                    own = __ldg(sw + i);
                }
                gather_rows<L, (L != 4)>(a, sw, beg, end, p);  // (L = 4: the masked tail cost G55 C3 3.6 %)
                d = (int)(end - beg);
            }
            if (a.do_cut && valid) {
                uint32_t g[L];
                cut_counts<L>(p, own, d, g);
                dsum += d;
                vc_add<L, CP>(C, g);
            }
            if (PBSA_BK_NIB && L <= 4) {
                // the 32 counts as nibbles (word k nibble j = trial 8k + j), so a
                // slot's count is one shared load and a shift; with L <= 3
                // (degree <= 7) the nibble holds raw + 7 = 2 p - d + 7 instead
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    uint32_t nib = 0;
#pragma unroll
                    for (int r = 0; r < L; ++r) {
                        uint32_t x = (p[r] >> (8 * k)) & 0xFFu;
                        x = (x | (x << 12)) & 0x000F000Fu;
                        x = (x | (x << 6)) & 0x03030303u;
                        x = (x | (x << 3)) & 0x11111111u;
                        nib |= x << r;
                    }
                    if (L <= 3) nib = (nib << 1) + (uint32_t)(7 - d) * 0x11111111u;
                    splane[k * 32 + lane] = nib;
                }
            } else {
#pragma unroll
                for (int r = 0; r < L; ++r) splane[r * 32 + lane] = p[r];
            }
            sown[lane] = own;
            sdeg[lane] = (uint32_t)d;
            snode[lane] = (uint32_t)i;
            sflip[lane] = 0;
            sexm[lane] = 0;
            mbar_wait_parity(mbar, parity);  // the staged records have landed
            __syncwarp();
            // 3. decisions of the fired slots (l, b): trial b's count from lane
            // l's planes, the draw, the prefilter; flips and undecided trials
            // go to lane l's masks (padding records are skipped)
            // branch-free so that a lane's four slots of a round interleave;
            // a padding record (~0) decides nothing (zero masks)
            auto fire_one = [&](uint4 rec, bool rec_in) {
                const bool real = rec.x != 0xFFFFFFFFu;
                const int b = (int)(rec.x & 31u), l = (int)((rec.x >> 5) & 31u);
                const int ii = (int)snode[l];
                int raw;
                if (PBSA_BK_NIB && L <= 3) {
                    raw = (int)((splane[(b >> 3) * 32 + l] >> (4 * (b & 7))) & 15u) - 7;
                } else if (PBSA_BK_NIB && L == 4) {
                    raw = 2 * (int)((splane[(b >> 3) * 32 + l] >> (4 * (b & 7))) & 15u) - (int)sdeg[l];
                } else {
                    int pop = 0;
#pragma unroll
                    for (int r = 0; r < L; ++r) pop |= (int)((splane[r * 32 + l] >> b) & 1u) << r;
                    raw = 2 * pop - (int)sdeg[l];
                }
                const float ir = a.i0f * (float)raw;
                uint32_t zh;
                if (NATIVE) {  // one Philox block per fired trial (fired trials are sparse)
                    uint32_t o[4];
                    philox4x32_10_rk((uint32_t)ii, count, a.ngroup + 8u * (uint32_t)w + (uint32_t)(b >> 2),
                                     kNativeTagR, a.rk, o);
                    zh = (b & 2) ? ((b & 1) ? o[3] : o[2]) : ((b & 1) ? o[1] : o[0]);
                } else {  // the record's first-absorb cache: only the second absorb remains
                    zh = packed_hash_hi_c(rec.z ^ count, rec.w);
                }
                __half2 pv;
                memcpy(&pv, &rec.y, 4);
                const uint32_t v = var_prefilter(pv, ir, zh, a.margin);
                const uint32_t bit = real ? 1u << b : 0u;
                if (rec_in && real) a.inp_out[((size_t)w * 32 + b) * a.n + ii] = __dmul_rn(a.i0, (double)raw);
                // (lane, flip bit, exact bit): the caller applies the masks
                // after a round's slots so their chains are not ordered by atomics
                return make_uint3((uint32_t)l, (v & 2u) ? 0u : (((v ^ (sown[l] >> b)) & 1u) ? bit : 0u),
                                  (v & 2u) ? bit : 0u);
            };
            auto apply = [&](uint3 m) {
                if (m.y) atomicOr(sflip + m.x, m.y);
                if (m.z) atomicOr(sexm + m.x, m.z);
            };
            const int Fe = F;
            if (a.inp_out == nullptr && Fe <= kBucketStage) {
                // four staged slots per lane and round (independent chains)
                // while at least 97 remain, then one per lane
                int j0 = 0;
                for (; PBSA_BK_ILP && j0 + 96 < Fe; j0 += 128) {
                    uint4 rec[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = j0 + 32 * u + lane;
                        rec[u] = j < Fe ? stage[j] : make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
                    }
                    uint3 m[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) m[u] = fire_one(rec[u], false);
#pragma unroll
                    for (int u = 0; u < 4; ++u) apply(m[u]);
                }
                for (; j0 < Fe; j0 += 32) {
                    const int j = j0 + lane;
                    if (j < Fe) apply(fire_one(stage[j], false));
                }
            } else {
                // past the staging list, or a launch recording inputs (last
                // sub-steps): slot j's segment from the table
                int sg = 0;
                for (int j = lane; j < Fe; j += 32) {
                    while ((int)pre[sg + 1] <= j) ++sg;
                    const uint4 rec = j < kBucketStage ? stage[j] : __ldg(src + beg16[sg] + (j - (int)pre[sg]));
                    apply(fire_one(rec, slast[sg] != 0));
                }
            }
            __syncwarp();
            if (valid) {
                uint32_t word = own ^ sflip[lane];
                const uint32_t ex = sexm[lane];
                if (ex) word = (word & ~ex) | var_exact_bits<L, NATIVE>(a, ex, p, d, w, i, count);
                a.snew[(size_t)w * a.n + i] = word;
            }
            __syncwarp();
            // (the staging list and tables are reused: order this tile's generic
            // reads before the next tile's bulk writes)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
    }
    if (a.do_cut)  // (the cut is taken on a cycle's first sub-step only)
        warp_cut_flush(C, dsum, lane, live ? a.pacc + (size_t)w * 32 : nullptr);
}

}  // namespace pbsa
