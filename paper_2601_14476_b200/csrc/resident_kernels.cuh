// resident_kernels.cuh -- resident cluster sweeps (one launch per run, state in shared
// memory): resident_sweep and resident_timing.  Instantiated per L in kernels_L*.cu.
#pragma once
#include "device_common.cuh"

namespace pbsa {

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
    uint16_t *adjS = reinterpret_cast<uint16_t *>(rowS + (per + 1));  // [rowptr[hi] - rowptr[lo]], 16-bit entries
    const uint32_t r0 = a.rowptr[lo], r1 = a.rowptr[hi];
    for (int k = tid; k <= hi - lo; k += blockDim.x) rowS[k] = a.rowptr[lo + k] - r0;
    for (uint32_t k = tid; k < r1 - r0; k += blockDim.x) adjS[k] = a.adj16[r0 + k];
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
                return cs[e & 0x7fffu] ^ (0u - (e >> 15));
            }, p);
            const int d = (int)(end - beg);
            uint32_t g[L];
            cut_counts<L>(p, own, d, g);
            dsum += d;
            vc_add<L, CP>(C, g);
            if (c == a.cycles) continue;  // final cut pass
            const uint32_t ui = (uint32_t)i;
            const uint2 *ctile = CACHED ? a.acache + ((size_t)w * a.chunks + (i >> 5)) * 1024 + cache_lane(i & 31) : nullptr;
            if (VARU) {  // the packed ALG=3 decision (sigmoid prefilter, exact recheck)
                const double i0 = a.i0[cc];
                const float i0f = (float)i0;
                const float2 *pr = a.prof + (size_t)w * 32 * a.n + i;
                uint32_t word = 0, exact = 0;
                uint32_t X[4];
                uint4 cpair = make_uint4(0u, 0u, 0u, 0u);  // CACHED: the current trial pair
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
                        const uint2 v = cache_get<true, true>(ctile, b, cpair);
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
                            philox4x32_10_rk(ui, count, grp + (uint32_t)(b >> 2), kNativeTagR, a.rk, X);
                        native_decide(X[b & 3], t, word);
                    } else if (CACHED) {
                        const uint2 v = cache_get<false, true>(ctile, b, cpair);
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
            uint4 cpair = make_uint4(0u, 0u, 0u, 0u);  // CACHED: the current trial pair
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
                    native_decide(X[b & 3], t, word);
                } else if (CACHED) {
                    const uint2 v = cache_get<false, true>(ctile, b, cpair);
                    tie = min(tie, packed_decide_n2(v.x ^ count, cache_c1(v.y), t, word));
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
    uint16_t *adjS = reinterpret_cast<uint16_t *>(rowS + per + 1);  // 16-bit entries
    for (int k = tid; k < a.n; k += blockDim.x) S0[k] = a.s_in[(size_t)w * a.n + k];
    if (tid < 32) key[tid] = a.kfc[(size_t)w * 32 + tid];
    const uint32_t r0 = a.rowptr[lo], r1 = a.rowptr[hi];
    for (int k = tid; k <= hi - lo; k += blockDim.x) rowS[k] = a.rowptr[lo + k] - r0;
    for (uint32_t k = tid; k < r1 - r0; k += blockDim.x) adjS[k] = a.adj16[r0 + k];
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
                return cs[e & 0x7fffu] ^ (0u - (e >> 15));
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

}  // namespace pbsa
