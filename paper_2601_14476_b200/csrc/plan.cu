// plan.cu -- plan creation: launch-shape choice, device uploads and tables (the
// reference loop being replaced is /root/reference/pkg/src/pbitsa/_kernels.py:68-175)
#include "runtime.h"

namespace pbsa_rt {

// Word-phase width for the packed sweep (W = one phase), from a wave model
// fitted on the C5 rows x 4096 (profiles/r02_summary.md, "phase width"): the
// launches of one phase hold phase_words x warps_per_word warps; the modelled
// throughput is (warps in flight / resident warps, at most 1) x (chunks /
// (warps x busiest warp's chunks)) x c/(c + 0.25) with c the chunks per warp (a
// launch's fixed cost per warp, ~190 instructions, is about a quarter of a
// chunk), x (l2_budget / cache)^0.35 for one phase whose hash cache (8 KiB per
// word and chunk) exceeds l2_budget; several phases must fit it.  l2_budget 0 allows one phase
// only.  *balance: spread the chunks over the fewest warps with the same
// busiest-warp count.
int64_t choose_phases(int64_t chunks, int64_t W, int64_t resident_warps, size_t l2_budget, bool *balance) {
    double best = -1;
    int64_t best_pw = W;
    *balance = false;
    const int64_t max_phases = l2_budget ? std::max<int64_t>(1, W / 4) : 1;
    for (int64_t nph = 1; nph <= max_phases; ++nph) {
        const int64_t pw = (W + nph - 1) / nph;
        if ((W + pw - 1) / pw != nph) continue;  // equal phases only
        const bool fits = (size_t)pw * (size_t)chunks * 8192 <= l2_budget;
        if (nph > 1 && !fits) continue;
        for (int bal = 0; bal < 2; ++bal) {
            int64_t wpw = std::min<int64_t>(std::max<int64_t>(1, resident_warps / pw), chunks);
            if (bal) {
                const int64_t per = (chunks + wpw - 1) / wpw;
                wpw = (chunks + per - 1) / per;
            }
            wpw = (wpw + pbsa::kPackedWarps - 1) / pbsa::kPackedWarps * pbsa::kPackedWarps;
            const int64_t per = (chunks + wpw - 1) / wpw;
            double eff = std::min(1.0, (double)(pw * wpw) / (double)resident_warps) * (double)chunks /
                         (double)(wpw * per) * (double)per / ((double)per + 0.25);
            if (!fits) eff *= std::pow((double)l2_budget / ((double)pw * (double)chunks * 8192.0), 0.35);
            if (eff > best + 1e-9) {
                best = eff;
                best_pw = pw;
                *balance = bal != 0;
            }
        }
    }
    return best_pw;
}



// Active-list setup for integer-valued models (see general_active).
void setup_active(pbsa_plan &P, int64_t n, const int64_t *indptr, const int64_t *indices,
                  const double *values, const double *hv, const double *lam, const double *delta,
                  const int64_t *period, int64_t pstride, int64_t trials, int64_t cycles,
                  int64_t t_res, int algo, int64_t alpha, double p_stall) {
    const int64_t nnz = indptr[n];
    int tshift = 0;
    while ((1LL << tshift) < P.Tp) ++tshift;
    if ((n << tshift) > (int64_t)UINT32_MAX || n * P.Tp > (int64_t)UINT32_MAX) return;
    for (int64_t k = 0; k < nnz; ++k)
        if (!is_integral(values[k])) return;
    cudaStream_t st = P.stream;
    std::vector<int32_t> vi(nnz), hi(n);
    bool any_h = false;
    int64_t rawmin = INT64_MAX, rawmax = INT64_MIN;
    for (int64_t i = 0; i < n; ++i) {
        hi[i] = (int32_t)hv[i];
        any_h |= hi[i] != 0;
        int64_t span = 0;
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) span += std::llabs((int64_t)values[k]);
        rawmin = std::min(rawmin, hi[i] - span);
        rawmax = std::max(rawmax, hi[i] + span);
    }
    if (rawmax - rawmin > (1LL << 30)) return;
    for (int64_t k = 0; k < nnz; ++k) vi[k] = (int32_t)values[k];
    P.vali.upload(vi, st);
    if (any_h) P.hi32.upload(hi, st);
    if (algo == 1) P.hist_i.alloc((size_t)n * alpha * trials);
    // table mode: plain rule (or a degenerate rule) with an ideal lam/delta
    bool ideal_ld = true;
    const int64_t prow = pstride ? trials : 1;
    if (lam)
        for (int64_t k = 0; k < prow * n && ideal_ld; ++k)
            ideal_ld = lam[k] == 1.0 && delta[k] == 0.0;
    const bool plain = algo == 0 || (algo == 1 && alpha == 1) || (algo == 2 && p_stall == 0.0);
    if (plain && ideal_ld && rawmax - rawmin < 65536) {
        P.rawmin = (int)rawmin;
        P.Kt = (int)(rawmax - rawmin + 1);
        std::vector<uint64_t> thr((size_t)cycles * P.Kt);
        for (int64_t c = 0; c < cycles; ++c)
            for (int64_t r = rawmin; r <= rawmax; ++r)
                thr[(size_t)c * P.Kt + (r - rawmin)] = threshold_h64(pb_libm_tanh(P.i0[c] * (double)r));
        P.athr.upload(thr, st);
    }
    // bucket every (trial, node) pair by its period; order inside a bucket is
    // node-major so neighbouring threads share CSR rows
    const int64_t maxcount = cycles * t_res;
    auto per_of = [&](int64_t t, int64_t i) -> int64_t {
        const int64_t pv = period ? period[(pstride ? t * n : 0) + i] : t_res;
        return std::min<int64_t>(pv, maxcount + 1);
    };
    std::vector<int64_t> bucket_of(maxcount + 2, -1), periods;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = 0; t < trials; ++t) {
            const int64_t pv = per_of(t, i);
            if (bucket_of[pv] < 0) {
                bucket_of[pv] = 0;
                periods.push_back(pv);
            }
        }
    std::sort(periods.begin(), periods.end());
    for (size_t b = 0; b < periods.size(); ++b) bucket_of[periods[b]] = (int64_t)b;
    std::vector<int64_t> bstart(periods.size() + 1, 0);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = 0; t < trials; ++t) ++bstart[bucket_of[per_of(t, i)] + 1];
    for (size_t b = 0; b < periods.size(); ++b) bstart[b + 1] += bstart[b];
    std::vector<uint32_t> list((size_t)bstart.back());
    std::vector<int64_t> fill(bstart.begin(), bstart.end() - 1);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = 0; t < trials; ++t)
            list[fill[bucket_of[per_of(t, i)]]++] = (uint32_t)((i << tshift) | t);
    P.alist.upload(list, st);
    // per active sub-step: descriptors of the buckets whose period divides the counter
    std::vector<int4> desc;
    int64_t maxtotal = 0;
    for (int64_t count = 0; count < maxcount; ++count) {
        pbsa_plan::ALaunch L{(uint32_t)count, count / t_res, (int64_t)desc.size(), 0, 0};
        int64_t cum = 0;
        for (size_t b = 0; b < periods.size(); ++b) {
            if (count % periods[b] != 0) continue;
            const int64_t len = bstart[b + 1] - bstart[b];
            desc.push_back(make_int4((int)bstart[b], (int)cum, (int)len, 0));
            cum += len;
        }
        L.ndesc = (int)(desc.size() - L.desc_off);
        if (L.ndesc > pbsa::kMaxActiveDesc) return;  // fall back to the full-pass kernel
        L.total = (int)cum;
        if (cum > 0) P.alaunch.push_back(L);
        maxtotal = std::max(maxtotal, cum);
    }
    P.adesc.upload(desc, st);
    P.st_g.alloc((size_t)maxtotal);
    P.st_v.alloc((size_t)maxtotal);
    // per-p-bit state in list order (coalesced per launch); per-trial profiles
    // are gathered into list order too
    const size_t Np = list.size();
    P.a_inputs.alloc(Np);
    P.a_counts.alloc(Np);
    if (lam && pstride) {
        std::vector<double> l(Np), d(Np);
        for (size_t li = 0; li < Np; ++li) {
            const int64_t i = list[li] >> tshift, t = list[li] & ((1u << tshift) - 1u);
            l[li] = lam[t * n + i];
            d[li] = delta[t * n + i];
        }
        P.lam.upload(l, st);
        P.delta.upload(d, st);
    }
    // fast mode for the plain rule: the draw folds like the packed path's
    // (i, count < 2^30), no per-p-bit state beyond the last inputs
    const bool plain_state_free = algo == 0 || (algo == 2 && p_stall == 0.0);
    const char *fenv = std::getenv("PBSA_ACTIVE_FAST");
    if (plain_state_free && n < (1LL << 30) && maxcount <= (1LL << 30) && !(fenv && fenv[0] == '0')) {
        P.fast = true;
        std::vector<uint64_t> krg(P.Tp);
        std::vector<uint2> kfc(P.Tp);
        for (int64_t t = 0; t < P.Tp; ++t) {
            krg[t] = P.kr_host[t] + kGamma;
            const uint32_t lo = (uint32_t)krg[t], hi = (uint32_t)(krg[t] >> 32);
            const uint32_t Y = hi ^ (hi >> 30);
            kfc[t] = make_uint2(lo ^ ((lo >> 30) | (hi << 2)), Y * 0x1CE4E5B9u);
        }
        P.krg.upload(krg, st);
        P.kfc.upload(kfc, st);
        if (lam && !P.athr.n) {
            if (pstride) {
                std::vector<float2> pf(Np);
                for (size_t li = 0; li < Np; ++li) {
                    const int64_t i = list[li] >> tshift, t = list[li] & ((1u << tshift) - 1u);
                    const double l = lam[t * n + i], d = delta[t * n + i];
                    pf[li] = make_float2((float)l, (float)(l * d));
                }
                P.aprof.upload(pf, st);
            } else {
                std::vector<float2> pf(n);
                for (int64_t i = 0; i < n; ++i) pf[i] = make_float2((float)lam[i], (float)(lam[i] * delta[i]));
                P.aprof.upload(pf, st);
            }
        }
        P.flips.alloc((size_t)std::max<int64_t>(maxtotal, 1));
        P.nflips.alloc(std::max<size_t>(P.alaunch.size(), 1));
        P.apcl.assign((size_t)trials * n, 0);
        for (int64_t t = 0; t < trials; ++t)
            for (int64_t i = 0; i < n; ++i) {
                const int64_t pv = per_of(t, i);
                P.apcl[(size_t)t * n + i] = (int32_t)pv;
                P.apmax = std::max(P.apmax, pv);
            }
        P.a_counts.release();
    }
    P.inputs.release();
    P.counts.release();
    P.tshift = tshift;
    P.tmask = (uint32_t)((1u << tshift) - 1u);
    P.active_mode = true;
    P.hist.release();  // the integer ring replaces the fp64 history
}

// Host-side forms of the per-trial key prefixes and of the packed path's
// per-trial constants and plain-rule threshold table (create_plan, and the
// per-call refresh of a cached one-shot plan).
void host_trial_keys(const uint64_t *keys, int64_t trials, int64_t Tp, std::vector<uint64_t> &kspin,
                     std::vector<uint64_t> &kr, std::vector<uint64_t> &kst) {
    kspin.assign(Tp, 0);
    kr.assign(Tp, 0);
    kst.assign(Tp, 0);
    for (int64_t t = 0; t < trials; ++t) {
        kspin[t] = habsorb(keys[t], 2);
        kr[t] = habsorb(keys[t], 3);
        kst[t] = habsorb(keys[t], 4);
    }
}

void host_packed_consts(const std::vector<uint64_t> &kr, std::vector<uint64_t> &krg, std::vector<uint2> &kfc) {
    krg.resize(kr.size());
    kfc.resize(kr.size());
    for (size_t t = 0; t < kr.size(); ++t) {
        krg[t] = kr[t] + kGamma;
        const uint32_t lo = (uint32_t)krg[t], hi = (uint32_t)(krg[t] >> 32);
        const uint32_t Y = hi ^ (hi >> 30);
        kfc[t] = make_uint2(lo ^ ((lo >> 30) | (hi << 2)), Y * 0x1CE4E5B9u);
    }
}

std::vector<uint64_t> host_plain_thresholds(const pbsa_plan &P) {
    // thresholds per (cycle, raw): inp = i0 * raw; act = r + tanh(inp) (lam = 1, delta = 0)
    // (native mode: the smallest Philox word X that gives +1, threshold_native)
    std::vector<uint64_t> thr((size_t)P.cycles * P.K);
    for (int64_t c = 0; c < P.cycles; ++c)
        for (int raw = -P.dmax; raw <= P.dmax; ++raw) {
            const double t = pb_libm_tanh(P.i0[c] * (double)raw);
            thr[(size_t)c * P.K + raw + P.dmax] = P.native ? threshold_native(t) : threshold_h64(t);
        }
    return thr;
}

void host_csr(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
              std::vector<uint32_t> &rowptr, std::vector<uint32_t> &adj32, std::vector<uint16_t> &adj16) {
    const int64_t nnz = indptr[n];
    rowptr.resize(n + 1);
    for (int64_t i = 0; i <= n; ++i) rowptr[i] = (uint32_t)indptr[i];
    // device CSR: 16-bit column | sign whenever n <= 32768 (the north_star
    // format, 2 bytes per coupling), 32-bit column | sign beyond
    adj16.clear();
    adj32.clear();
    if (n <= 32768) {
        adj16.resize(nnz);
        for (int64_t k = 0; k < nnz; ++k)
            adj16[k] = (uint16_t)((uint32_t)indices[k] | (values[k] < 0 ? 0x8000u : 0u));
    } else {
        adj32.resize(nnz);
        for (int64_t k = 0; k < nnz; ++k)
            adj32[k] = (uint32_t)indices[k] | (values[k] < 0 ? 0x80000000u : 0u);
    }
}

// Packed path with a varied profile: the fp32 / fp16 prefilter pairs and the
// exact fp64 profile on the device, and with a timing spread the bit-sliced
// clamped periods, their class table and the launch list of every sub-step
// some present period divides (_kernels.py:110-127).
void packed_variability_setup(pbsa_plan &P, int64_t n, int64_t trials, int64_t cycles, int64_t t_res,
                              const double *lam, const double *delta, const int64_t *period, int64_t pstride,
                              bool native_prof, cudaStream_t st) {
    const int64_t maxcount = cycles * t_res;
    std::vector<uint8_t> divs;
    // per-p-bit profile, trial-major [Tp][n] (padding trials: ideal).  The
    // fp32 pair of the timing kernels is [W][n][32] instead: their fired
    // p-bits are a sparse random ~15 % of each (word, node), so keeping a
    // node's 32 trials in 256 contiguous bytes lets nearby fires share
    // DRAM bursts that the [W][32][n] layout spreads over 32 rows
    const int64_t Tp = P.Tp;
    const bool node_major = !P.var_uniform;
    if (!native_prof && pstride == n) {
        // per-trial rows already in the plan's [trial][node] layout: upload
        // the exact profile as given (padding rows ideal) and round the
        // prefilter pairs on the device (no host copies or conversion)
        P.lam64.alloc((size_t)Tp * n);
        P.del64.alloc((size_t)Tp * n);
        CK(cudaMemcpyAsync(P.lam64.p, lam, (size_t)trials * n * sizeof(double), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(P.del64.p, delta, (size_t)trials * n * sizeof(double), cudaMemcpyHostToDevice, st));
        P.lam64.bytes_up = P.del64.bytes_up = (size_t)trials * n * sizeof(double);
        if (Tp > trials) {
            pbsa::fill_f64<<<grid_for((Tp - trials) * n, 256), 256, 0, st>>>(
                P.lam64.p + (size_t)trials * n, (Tp - trials) * n, 1.0);
            CK(cudaMemsetAsync(P.del64.p + (size_t)trials * n, 0, (size_t)(Tp - trials) * n * sizeof(double), st));
        }
    }
    if (native_prof || pstride == n) {  // pairs from the device copy of the exact profile
        if (node_major) P.prof16.alloc((size_t)Tp * n); else P.prof.alloc((size_t)Tp * n);
        pbsa::profile_pairs<<<grid_for(Tp * n, 256), 256, 0, st>>>(
            P.lam64.p, P.del64.p, Tp, (int)n, node_major ? P.prof16.p : nullptr,
            node_major ? nullptr : P.prof.p);
        CK(cudaGetLastError());
    } else {
        std::vector<float2> pf(node_major ? 0 : (size_t)Tp * n, make_float2(1.0f, 0.0f));
        std::vector<__half2> pf16(node_major ? (size_t)Tp * n : 0, __floats2half2_rn(1.0f, 0.0f));
        std::vector<double> l64((size_t)Tp * n, 1.0), d64((size_t)Tp * n, 0.0);
        parallel_for(trials, 16, [&](int64_t t0, int64_t t1) {
            for (int64_t t = t0; t < t1; ++t)
                for (int64_t i = 0; i < n; ++i) {
                    const size_t src = (size_t)(pstride ? t * n : 0) + i, dst = (size_t)t * n + i;
                    const size_t pdst = node_major ? ((size_t)(t >> 5) * n + i) * 32 + (t & 31) : dst;
                    l64[dst] = lam[src];
                    d64[dst] = delta[src];
                    // timing kernels: fp16 pair (overflow -> inf -> the exact recheck)
                    if (node_major)
                        pf16[pdst] = __floats2half2_rn((float)lam[src], (float)(lam[src] * delta[src]));
                    else
                        pf[pdst] = make_float2((float)lam[src], (float)(lam[src] * delta[src]));
                }
        });
        if (node_major) P.prof16.upload(pf16, st); else P.prof.upload(pf, st);
        P.lam64.upload(l64, st);
        P.del64.upload(d64, st);

    }
    P.inp_var.alloc((size_t)Tp * n);
    if (!P.var_uniform) {
        // clamped periods (a period >= cycles * t_res fires only at count 0),
        // bit-sliced per word: plane k bit b = bit k of trial 32w+b's period
        P.nplanes = 1;
        while ((1LL << P.nplanes) <= P.pmax) ++P.nplanes;
        if (!native_prof) P.pcl.assign((size_t)trials * n, 0);
        std::vector<uint32_t> planes((size_t)P.W * P.nplanes * n, 0u);
        parallel_for(P.W, 1, [&](int64_t w0, int64_t w1) {
            for (int64_t w = w0; w < w1; ++w)
                for (int b = 0; b < 32; ++b) {
                    const int64_t t = w * 32 + b;
                    for (int64_t i = 0; i < n; ++i) {
                        int64_t pc = t_res;
                        if (t < trials && native_prof) {
                            pc = P.pcl[(size_t)t * n + i];
                        } else if (t < trials) {
                            pc = std::min<int64_t>(period[(pstride ? t * n : 0) + i], maxcount);
                            P.pcl[(size_t)t * n + i] = (uint8_t)pc;
                        }
                        for (int k = 0; k < P.nplanes; ++k)
                            planes[((size_t)w * P.nplanes + k) * n + i] |= (uint32_t)((pc >> k) & 1) << b;
                    }
                }
        });
        P.pplanes.upload(planes, st);
        std::vector<char> present(256, 0);
        for (uint8_t pc : P.pcl) present[pc] = 1;  // (padding trials never matter)
        std::vector<uint8_t> lut(256, 0), cdivs, cper;
        for (int pc = 1; pc < 256; ++pc)
            if (present[pc]) {
                lut[pc] = (uint8_t)P.nclass++;
                cper.push_back((uint8_t)pc);
            }
        P.blut.upload(lut, st);
        P.bcper.upload(cper, st);
        // ... or, with a timing spread, every sub-step some present period
        // divides (the first sub-step of each cycle always runs: it takes the cut)
        for (int64_t c = 0; c < cycles; ++c)
            for (int64_t s = 0; s < t_res; ++s) {
                const int64_t count = c * t_res + s;
                const int64_t off = (int64_t)divs.size();
                for (int64_t pc = 1; pc <= P.pmax; ++pc)
                    if (present[pc] && count % pc == 0) {
                        divs.push_back((uint8_t)pc);
                        cdivs.push_back(lut[pc]);
                    }
                const int nd = (int)((int64_t)divs.size() - off);
                if (nd > pbsa::kMaxDivisors) fail(PBSA_EINVAL, "too many dividing periods");
                P.max_ndiv = std::max(P.max_ndiv, nd);
                if (s == 0 || nd > 0)
                    P.plaunch.push_back({(uint32_t)count, c, s == 0, nd, off, true,
                                         count >= maxcount - P.pmax});
            }
        if (divs.empty()) {
            divs.push_back(0);
            cdivs.push_back(0);
        }
        P.vdivs.upload(divs, st);
        P.bdivs.upload(cdivs, st);
    }
}

// Launch shape of the packed sweep: word phases (choose_phases), the
// first-absorb hash cache, warps per word, chains of word groups.
void packed_launch_shape(pbsa_plan &P, int device, int64_t n, int64_t dmax) {
    // launch shape: one wave of resident warps, each owning one word
    // cache the sub-step-independent first absorb of every (trial, node)
    // draw when it fits the budget (PBSA_PACKED_CACHE=0/1 overrides)
    // phase width in words (PBSA_PACKED_PHASE_WORDS overrides; 0 = all)
    // Large batches run in word phases whose hash cache stays L2-resident
    // across their cycles (G81: 13 words, ~67 MB), which keeps HBM (and the
    // 1 kW power cap) out of the loop.  The width comes from a wave model
    // (choose_phases): fill the resident warps, give every warp the same
    // chunk count, keep that count >= 2, fit the phase's cache in 5/8 of L2.
    // A timing spread multiplies the launches by t_res: one phase, four chains.
    const bool many_launches = P.var_mode && !P.var_uniform;
    int sm_count = 148, l2_bytes = 0;
    CK(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device));
    CK(cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, device));
    // (SpSA streams its per-p-bit drive index, which no phase keeps in L2: unphased)
    // (native Philox draws keep no cache, so nothing gains from phases: measured
    // G81 x 4096 9.1e11 updates/s unphased vs 7.8e11 in phases of 13)
    const bool may_phase = !g_oneshot && !many_launches && !P.spsa_packed && !P.native;
    const size_t smem = (size_t)std::max(P.K, (P.dmax + 1) * 32) * 8 + 512 + 2 * pbsa::kPackedWarps * 32 * 8 + 16 +
                         pbsa::kPackedFlushBytes;
    const size_t smem_up = many_launches ? pbsa::kTimingSmem : smem;
    int occ = 0;
    {
        // (the kernel instance, so its occupancy, does not depend on the phase width)
        PackedKernel k0 = packed_kernel_for(P.L, true, !many_launches && !P.native, P.tapsa_packed, P.spsa_packed,
                                            P.var_mode ? (P.var_uniform ? 1 : 2) : 0, P.native);
        set_packed_smem(k0, smem_up);
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k0, pbsa::kPackedThreads, smem_up));
        occ = std::max(occ, 1);
    }
    P.chunks = (int)((n + 31) / 32);
    bool balance_chunks = false;
    P.phase_words = choose_phases(P.chunks, P.W, (int64_t)sm_count * occ * pbsa::kPackedWarps,
                                  may_phase ? (size_t)l2_bytes * 5 / 8 : 0, &balance_chunks);
    if (P.phase_words >= P.W) P.phase_words = 0;
    // one-shot calls of the plain rule on the launched path run pipelined
    // (PBSA_PIPELINE=0 disables): four word phases, each phase's outputs
    // copied back while the next anneals (decided again below once the
    // resident choice is known)
    P.pipelined = (g_oneshot || g_cached_oneshot) && !many_launches && !P.var_mode && !P.tapsa_packed &&
                  !P.spsa_packed && !P.tapsa_hist_from_raw && P.W >= 16;
    if (const char *env = std::getenv("PBSA_PIPELINE")) P.pipelined = P.pipelined && env[0] != '0';
    // a cached one-shot plan keeps the benchmark's phases and chains (its
    // launches are replayed from a graph, so their count costs nothing)
    P.capturing_outputs = g_cached_oneshot && P.pipelined;
    // (up to four phases, but each phase at least two waves of word-warps:
    // measured G81 x 512 one-shot, four phases of 4 words 36.6 ms)
    // a cached one-shot plan of an unphased batch still splits it in two when
    // each half fills two waves of word-warps: the second half's outputs are
    // then the only ones left to copy after the anneal
    if (P.capturing_outputs && (P.phase_words == 0 || P.phase_words >= P.W)) {
        const int64_t fill = ((int64_t)sm_count * 32 + (n + 31) / 32 - 1) / ((n + 31) / 32);
        if (P.W >= 4 * fill) P.phase_words = (P.W + 1) / 2;  // (measured: halves of one wave lose)
    }
    if (P.pipelined && !P.capturing_outputs) {
        const int64_t fill = (2LL * sm_count * 32 + (n + 31) / 32 - 1) / ((n + 31) / 32);
        P.phase_words = std::min<int64_t>(P.W, std::max<int64_t>((P.W + 3) / 4, fill));
    }
    if (const char *env = std::getenv("PBSA_PACKED_PHASE_WORDS")) P.phase_words = std::atoi(env);
    if (const char *env = std::getenv("PBSA_PDL")) P.use_pdl = env[0] != '0';
    if (P.phase_words <= 0 || P.phase_words > P.W) P.phase_words = P.W;
    const size_t cache_entries = (size_t)P.phase_words * ((n + 31) / 32) * 1024;
    // (with a timing spread the fired trials of a word are sparse: no cache)
    P.use_cache = cache_entries * 8 <= (32ULL << 30) && !many_launches;
    if (const char *env = std::getenv("PBSA_PACKED_CACHE")) P.use_cache = env[0] == '1' && !many_launches;
    if (P.native) P.use_cache = false;  // Philox draws cache nothing
    if (P.use_cache) P.acache.alloc(cache_entries);
    PackedKernel kern = packed_kernel_for(P.L, true, P.use_cache, P.tapsa_packed, P.spsa_packed,
                                          P.var_mode ? (P.var_uniform ? 1 : 2) : 0, P.native);
    set_packed_smem(kern, smem_up);
    set_packed_smem(packed_kernel_for(P.L, false, false), smem);
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, pbsa::kPackedThreads, smem_up));
    occ = std::max(occ, 1);
    const int64_t target_warps = (int64_t)sm_count * occ * pbsa::kPackedWarps;
    int64_t wpw = std::max<int64_t>(1, target_warps / P.phase_words);  // one phase at a time
    wpw = std::min<int64_t>(wpw, P.chunks);
    // equal chunk counts per warp: a launch lasts as long as its busiest
    // warp, so spread the chunks over the fewest warps that give the same
    // maximum, when choose_phases scores that higher (PBSA_BALANCE_CHUNKS=0/1)
    {
        bool balance = balance_chunks;
        if (const char *env = std::getenv("PBSA_BALANCE_CHUNKS")) balance = env[0] != '0';
        if (balance) {
            const int64_t per = (P.chunks + wpw - 1) / wpw;
            wpw = (P.chunks + per - 1) / per;
        }
    }
    // the per-thread bit-sliced cut counter holds sum(degree) < 2^(L+2)
    const int64_t cap = (1LL << (P.L + 2)) - 1, dm = std::max<int64_t>(dmax, 1);
    if (dm > cap) fail(PBSA_EINVAL, "degree too large for the packed cut counter");
    const int64_t max_tasks = cap / dm;  // chunks one warp may take
    wpw = std::max<int64_t>(wpw, std::min<int64_t>((P.chunks + max_tasks - 1) / max_tasks, P.chunks));
    // a multiple of the block's warps, so each block works on one word and
    // reduces the cut once (PBSA_CTA_FLUSH=0 keeps one flush per warp)
    P.cta_flush = true;
    if (const char *env = std::getenv("PBSA_CTA_FLUSH")) P.cta_flush = env[0] != '0';
    if (P.cta_flush) wpw = (wpw + pbsa::kPackedWarps - 1) / pbsa::kPackedWarps * pbsa::kPackedWarps;
    if (const char *env = std::getenv("PBSA_WARPS_PER_WORD"))  // (experiments; bounded like the default)
        wpw = std::max<int64_t>(std::min<int64_t>(std::atoi(env), P.chunks),
                                (P.chunks + max_tasks - 1) / max_tasks);
    P.warps_per_word = (int)wpw;
    // concurrent chains of word groups (PBSA_PACKED_CHAINS overrides; 1 disables)
    // small batches need many chains to hide launch gaps; large ones only a
    // couple (fewer graph nodes to instantiate)
    int chains = (many_launches || (P.spsa_packed && !g_oneshot && P.W >= 64)) ? 4
                                                                 : (int)std::max<int64_t>(1, std::min<int64_t>(16, 256 / P.phase_words));
    if (P.pipelined && !P.capturing_outputs) chains = 2;  // launched directly: keep the launch count low
    if (const char *env = std::getenv("PBSA_PACKED_CHAINS")) chains = std::max(1, std::atoi(env));
    chains = (int)std::min<int64_t>(chains, P.W);
    if (chains > 1) CK(cudaEventCreateWithFlags(&P.ev_fork, cudaEventDisableTiming));
    for (int g = 1; g < chains; ++g) {
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        P.chain_streams.push_back(cs);
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        P.ev_join.push_back(e);
    }
    P.packed_blocks = (int)grid_for(P.W * wpw, pbsa::kPackedWarps);
}

// Resident cluster kernels for small batches of small dense graphs: a
// word's double-buffered state in shared memory, one launch per run.
void resident_setup(pbsa_plan &P, int device, int64_t n, const int64_t *indptr, int64_t alpha, int64_t cycles,
                    cudaStream_t st) {
    const int64_t nnz = indptr[n];
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    // resident mode (plain rule, ideal profile): a word's double-buffered
    // state in shared memory; cluster size so that W clusters cover the SMs
    {
        const bool plain = !P.tapsa_packed && !P.spsa_packed && !P.var_mode;
        const bool timing = P.var_mode && !P.var_uniform;
        const bool varu = P.var_mode && P.var_uniform;
        const bool tap = P.tapsa_packed && !P.var_mode;
        const int tab = tap ? P.K : (P.L <= 4 ? (P.dmax + 1) * 16 : P.K);
        P.res_smem = 512 + 2 * (size_t)tab * 8 + 32 * 8 + 8 * (size_t)n;  // two tables
        int max_smem = 0;
        CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        // measured: small batches (<= 64 words) of small dense graphs (n <= 2500,
        // mean degree >= 8: G1, G47, G22) run 1.1-2.2x faster resident; sparse
        // or larger problems are faster with launched sweeps
        // (TApSA: the launched sweep re-reads the ring every cycle; resident wins to
        // 128 words: G1 x 4096 alpha 4 27.2 -> 20.5 ms, G47 18.2 -> 16.5, G22 even)
        // (round 2, after the launched sweeps' instruction trims: resident up to 32
        // words, 64 at mean degree >= 32.  Timing spread vs the period-bucket
        // kernel, 300 cycles: resident G1 x 1024 / 2048 16 / 33 ms vs 37 / 41, G22
        // x 1024 20 vs 28; bucket G22 x 2048 / 4096 33 / 61 vs 41 / 70, G47 x 2048 /
        // 4096 27 / 32 vs 30 / 40.  Plain rule, 1000 cycles: resident G1 x 2048
        // 11.0 vs 13.9 ms, G22 x 1024 7.7 vs 8.7; launched G22 x 2048 11.2 vs 14.9)
        const bool small = P.W <= 32 || (P.W <= 64 && nnz >= 32 * n);
        bool want = (small || (P.tapsa_packed && !P.var_mode && P.W <= 128)) && n <= 2500 && nnz >= 8 * n;
        if (const char *env = std::getenv("PBSA_RESIDENT")) want = env[0] == '1';
        want = want && n <= 32768;  // (the resident kernels stage the 16-bit CSR)
        int csz = 1;  // (measured: 8 for a handful of words, 4 beats 8 at 32 words)
        while (csz < (P.W <= 8 ? 8 : 4) && P.W * csz < sms) csz *= 2;
        if (const char *env = std::getenv("PBSA_RESIDENT_CS")) csz = std::max(1, std::atoi(env));
        const int64_t per = (n + csz - 1) / csz;
        int64_t slice = 0;  // largest CTA slice of the adjacency
        for (int64_t r = 0; r < csz; ++r) {
            const int64_t lo = std::min<int64_t>(n, r * per), hi = std::min<int64_t>(n, lo + per);
            slice = std::max<int64_t>(slice, indptr[hi] - indptr[lo]);
        }
        P.res_smem += 4 * (size_t)(per + 1) + 2 * (size_t)slice + 4;  // (16-bit CSR slice)
        if (tap) P.res_smem += 4 * (size_t)alpha * P.L * per;  // the ring slice
        if (timing) {
            // two lanes per node when a CTA's slice still takes one pass of <= 16 warps
            // (measured: G1 C2 sigma_nu 1.0 70 -> 63 ms; a second pass costs more: G22)
            P.res_split = (per + 15) / 16 <= 16;
            if (const char *env = std::getenv("PBSA_RES_SPLIT")) P.res_split = env[0] == '1';
            const int64_t thr = std::min<int64_t>(512, P.res_split ? ((per + 15) / 16) * 32 : ((per + 31) / 32) * 32);
            P.res_smem = 32 * 8 + 8 * (size_t)n + (thr / 32) * (256 + 4096) + pbsa::kMaxDivisors * 32 +
                         4 * (size_t)(P.nplanes * per + per + 1) + 2 * (size_t)slice + 68;
            // stage the CTA's fp16 profile slice too when it fits (PBSA_RES_PROF=0 disables)
            const size_t prof_bytes = 4 * (size_t)per * 32;
            const char *penv = std::getenv("PBSA_RES_PROF");
            P.res_prof_smem = (!penv || penv[0] != '0') && P.res_smem + prof_bytes <= (size_t)max_smem;
            if (P.res_prof_smem) P.res_smem += prof_bytes;
        }
        // (per-thread cut counters take up to 32 nodes: 16 warps x 16 nodes x 32)
        if (timing && want && P.res_smem <= (size_t)max_smem && per <= 16 * 16 * 32) {
            P.resident = true;
            P.res_timing = true;
            P.res_cs = csz;
            P.res_threads = (int)std::min<int64_t>(512, P.res_split ? ((per + 15) / 16) * 32 : ((per + 31) / 32) * 32);
            std::vector<pbsa::RLaunch> rl;
            for (const pbsa_plan::PLaunch &pl : P.plaunch)
                rl.push_back({pl.count, (int)pl.cycle, pl.do_cut, pl.ndiv, (int)pl.div_off, pl.inp ? 1 : 0,
                              P.i0[std::min<int64_t>(pl.cycle, cycles - 1)]});
            P.rlaunch.upload(rl, st);
            if (!P.i0_dev.n) P.i0_dev.upload(P.i0, st);
            ResidentTimingKernel rk = resident_timing_for(P.L, P.native);
            CK(cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.res_smem));
            if (csz > 8) CK(cudaFuncSetAttribute(rk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        } else if ((plain || varu || tap) && want && P.res_smem <= (size_t)max_smem && per <= 32 * 512) {
            // (the per-thread cut counter takes up to 32 nodes)
            const int thr = (int)std::min<int64_t>(512, ((per + 31) / 32) * 32);
            P.resident = true;
            P.res_cs = csz;
            P.res_threads = thr;
            if (P.use_cache && P.phase_words < P.W) P.acache.alloc((size_t)P.W * P.chunks * 1024);
            P.phase_words = P.W;
            P.res_tapsa = tap;
            ResidentKernel rk = resident_kernel_for(P.L, P.use_cache, varu, P.native, tap);
            CK(cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.res_smem));
            if (varu && !P.i0_dev.n) P.i0_dev.upload(P.i0, st);
            if (csz > 8) CK(cudaFuncSetAttribute(rk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
    }
    if (P.resident) P.pipelined = P.capturing_outputs = false;
}

// Launched path: degree-sorted processing order of irregular graphs, and
// the period-bucket slot records of a timing spread.
void order_and_bucket_setup(pbsa_plan &P, int64_t n, const int64_t *indptr, cudaStream_t st) {
    const int64_t nnz = indptr[n];
    const bool many_launches = P.var_mode && !P.var_uniform;
    // irregular graphs on the launched path: warps take nodes in degree
    // order, so a chunk's lanes have similar degrees and the gather loop
    // runs ~ their degree, not the largest of 32 random ones (labels, spin
    // layout and draws are unchanged; PBSA_DEGREE_ORDER=0/1 overrides)
    if (!P.resident && !P.reg4) {
        std::vector<uint32_t> ord(n);
        for (int64_t i = 0; i < n; ++i) ord[i] = (uint32_t)i;
        std::stable_sort(ord.begin(), ord.end(), [&](uint32_t x, uint32_t y) {
            return indptr[x + 1] - indptr[x] > indptr[y + 1] - indptr[y];
        });
        double sum_max = 0, sum_deg = (double)nnz;
        for (int64_t c0 = 0; c0 < n; c0 += 32) {
            int64_t mx = 0;
            for (int64_t i = c0; i < std::min<int64_t>(n, c0 + 32); ++i)
                mx = std::max<int64_t>(mx, indptr[i + 1] - indptr[i]);
            sum_max += (double)mx * (double)(std::min<int64_t>(n, c0 + 32) - c0);
        }
        // (measured, 1024 trials: sparse random graphs gain -- G55 12.6 -> 11.0 ms, G60
        // 15.1 -> 13.1 ms -- while dense ones lose to the scattered own-word and
        // spin-store accesses -- G22 9.0 -> 10.9 ms, G1 12.2 -> 13.6 ms)
        bool want = sum_max > 1.15 * sum_deg && nnz < 8 * n;
        if (const char *env = std::getenv("PBSA_DEGREE_ORDER")) want = env[0] == '1';
        if (want) {
            ord.resize((size_t)P.chunks * 32, (uint32_t)n);
            P.order.upload(ord, st);
        }
    }
    // timing spread on the launched path: sort every tile's slots into
    // period buckets once (PBSA_BUCKET=0 keeps packed_sweep_timing)
    if (many_launches && !P.resident && P.max_ndiv <= pbsa::kBucketMaxDiv) {
        const char *benv = std::getenv("PBSA_BUCKET");
        P.bucket = !benv || benv[0] != '0';
    }
    if (P.bucket) {
        const size_t tiles = (size_t)P.W * P.chunks;
        P.brec.alloc(tiles * 1024);
        P.boff.alloc(tiles * (P.nclass + 1));
        pbsa::bucket_build<<<grid_for((int64_t)tiles, 8), 256, 0, st>>>(
            P.pplanes.p, P.nplanes, P.blut.p, P.prof16.p, P.krg.p, (int)n, P.chunks, (int)P.W,
            P.nclass, P.brec.p, P.boff.p, P.order.n ? P.order.p : nullptr);
        CK(cudaGetLastError());
        P.prof16.drop();   // (the slot-ordered copy replaces them)
        P.pplanes.drop();
        const PackedKernel bk = bucket_kernel_for(P.L, P.native);
        set_packed_smem(bk, pbsa::bucket_smem_bytes(P.L));
        int bocc = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bocc, bk, pbsa::kPackedThreads,
                                                         pbsa::bucket_smem_bytes(P.L)));
        (void)bocc;
    }
}

void create_plan(pbsa_plan &P, int device, int64_t n, const int64_t *indptr,
                 const int64_t *indices, const double *values, const double *hv, int64_t mm,
                 const int64_t *mei, const int64_t *mej, const double *mew, int64_t gm,
                 const int64_t *gei, const int64_t *gej, const int64_t *gew, const double *lam,
                 const double *delta, const int64_t *period, int64_t pstride, double i0_min,
                 double beta, int64_t cycles, int64_t t_res, int algo, int64_t alpha,
                 double p_stall, int64_t trials, const uint64_t *keys, int rng_mode,
                 uint64_t rng_seed, int64_t first_trial, const double *native_sig) {
    // ------------------------------------------------------- validation
    if (rng_mode != PBSA_RNG_REPLAY && rng_mode != PBSA_RNG_PHILOX)
        fail(PBSA_EINVAL, "rng_mode must be 0 (replay) or 1 (philox)");
    if (rng_mode == PBSA_RNG_PHILOX && (first_trial < 0 || first_trial % 4 != 0 ||
                                        first_trial + trials + 31 >= (1LL << 33)))
        fail(PBSA_EINVAL, "philox mode: first_trial must be a multiple of 4 in [0, 2^33)");
    if (n < 1 || n > INT32_MAX / 2) fail(PBSA_EINVAL, "n must be in [1, 2^30), got %lld", (long long)n);
    if (trials < 1 || trials > (1LL << 24)) fail(PBSA_EINVAL, "trials must be in [1, 2^24]");
    if (cycles < 1) fail(PBSA_EINVAL, "cycles must be >= 1");
    if (t_res < 1) fail(PBSA_EINVAL, "t_res must be >= 1");
    if (cycles * t_res >= (1LL << 31)) fail(PBSA_EINVAL, "cycles * t_res must be < 2^31");
    if (algo < 0 || algo > 2) fail(PBSA_EINVAL, "algo must be 0 (psa), 1 (tapsa) or 2 (spsa)");
    if (alpha < 1 || alpha > 4096) fail(PBSA_EINVAL, "alpha must be in [1, 4096]");
    if (!(p_stall >= 0.0 && p_stall <= 1.0)) fail(PBSA_EINVAL, "p_stall must lie in [0, 1]");
    if (!(i0_min > 0.0) || !(beta > 0.0)) fail(PBSA_EINVAL, "i0_min and beta must be > 0");
    if (!indptr || !hv || !keys) fail(PBSA_EINVAL, "null model/keys pointer");
    if (indptr[n] > 0 && (!indices || !values)) fail(PBSA_EINVAL, "null CSR pointer");
    if ((mm > 0 && (!mei || !mej || !mew)) || (gm > 0 && (!gei || !gej || !gew)))
        fail(PBSA_EINVAL, "null edge pointer");
    if (pstride != 0 && pstride != n) fail(PBSA_EINVAL, "profile_stride must be 0 or n");
    if ((lam == nullptr) != (delta == nullptr) || (lam == nullptr) != (period == nullptr))
        fail(PBSA_EINVAL, "lam, delta and period must all be given or all be NULL");
    const bool native_prof = native_sig && (native_sig[0] != 0.0 || native_sig[1] != 0.0 || native_sig[2] != 0.0);
    if (native_sig) {
        if (lam) fail(PBSA_EINVAL, "native profiles take sigmas, not lam/delta/period arrays");
        if (rng_mode != PBSA_RNG_PHILOX) fail(PBSA_EINVAL, "native profiles need rng_mode=philox");
        for (int k = 0; k < 3; ++k)
            if (!(std::isfinite(native_sig[k]) && native_sig[k] >= 0.0))
                fail(PBSA_EINVAL, "native profile sigmas must be finite and >= 0");
    }
    if (indptr[0] != 0) fail(PBSA_EINVAL, "indptr[0] must be 0");
    for (int64_t i = 0; i < n; ++i)
        if (indptr[i + 1] < indptr[i]) fail(PBSA_EINVAL, "indptr must be non-decreasing");
    const int64_t nnz = indptr[n];
    if (nnz >= (1LL << 31)) fail(PBSA_EINVAL, "too many couplings");
    for (int64_t k = 0; k < nnz; ++k)
        if (indices[k] < 0 || indices[k] >= n) fail(PBSA_EINVAL, "CSR index out of range");
    for (int64_t k = 0; k < mm; ++k)
        if (mei[k] < 0 || mei[k] >= n || mej[k] < 0 || mej[k] >= n)
            fail(PBSA_EINVAL, "model edge out of range");
    for (int64_t k = 0; k < gm; ++k)
        if (gei[k] < 0 || gei[k] >= n || gej[k] < 0 || gej[k] >= n)
            fail(PBSA_EINVAL, "graph edge out of range");
    const int64_t prow = pstride ? trials : 1;
    if (period)
        for (int64_t k = 0; k < prow * n; ++k)
            if (period[k] < 1) fail(PBSA_EINVAL, "period entries must be >= 1");

    P.device = device;
    P.n = n;
    P.T = trials;
    P.W = (trials + 31) / 32;
    P.Tp = P.W * 32;
    P.cycles = cycles;
    P.t_res = t_res;
    P.algo = algo;
    P.alpha = alpha;
    P.p_stall = p_stall;
    P.nnz = nnz;
    P.has_graph = gm > 0;
    // prefilter margin scale (tests: huge sends every update to the exact recheck)
    if (const char *env = std::getenv("PBSA_VAR_MARGIN")) P.var_margin = (float)std::atof(env);

    P.i0.resize(cycles);
    {
        double x = i0_min;  // repeated division, as run (_kernels.py:118, 172-173)
        for (int64_t c = 0; c < cycles; ++c) {
            P.i0[c] = x;
            if (c < cycles - 1) x = x / beta;
        }
    }

    DeviceGuard dg(device);
    CK(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
    P.stream_holder.s = P.stream;
    raise_pool_threshold(device);
    AllocStream as(P.stream);
    for (cudaEvent_t *e : {&P.ev_start, &P.ev_sweep0, &P.ev_sweep1, &P.ev_end}) CK(cudaEventCreate(e));
    cudaStream_t st = P.stream;

    // native profiles: drawn on the device (lam, delta fp64 [Tp][n] straight into
    // the plan's exact-recheck buffers); the clamped periods come back to the
    // host, which plans the sub-step launches and the period buckets from them
    int64_t native_pmax = 0;
    bool native_overflow = false;
    if (native_prof) {
        P.lam64.alloc((size_t)P.Tp * n);
        P.del64.alloc((size_t)P.Tp * n);
        DevBuf<uint8_t> pcl_dev;
        pcl_dev.alloc((size_t)P.Tp * n);
        DevBuf<int> ovf;
        ovf.alloc(1);
        CK(cudaMemsetAsync(ovf.p, 0, sizeof(int), st));
        pbsa::native_profiles<<<grid_for(P.Tp * n, 256), 256, 0, st>>>(
            (uint32_t)rng_seed, (uint32_t)(rng_seed >> 32), (uint64_t)first_trial, trials, P.Tp, (int)n,
            (int)t_res, native_sig[0], native_sig[1], native_sig[2], cycles * t_res, P.lam64.p, P.del64.p,
            pcl_dev.p, ovf.p);
        CK(cudaGetLastError());
        P.pcl.resize((size_t)trials * n);
        int ov = 0;
        CK(cudaMemcpyAsync(P.pcl.data(), pcl_dev.p, P.pcl.size(), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&ov, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        native_overflow = ov != 0;
        for (uint8_t pc : P.pcl) native_pmax = std::max<int64_t>(native_pmax, pc);
    }

    // --------------------------------------------------- path selection
    bool unit_J = true, zero_h = true;
    int64_t dmax = 0;
    for (int64_t k = 0; k < nnz; ++k)
        if (values[k] != 1.0 && values[k] != -1.0) { unit_J = false; break; }
    for (int64_t i = 0; i < n; ++i) {
        if (hv[i] != 0.0) zero_h = false;
        dmax = std::max<int64_t>(dmax, indptr[i + 1] - indptr[i]);
    }
    bool ideal = !native_prof;
    if (lam) {
        for (int64_t k = 0; k < prow * n && ideal; ++k)
            if (lam[k] != 1.0 || delta[k] != 0.0 || period[k] != t_res) ideal = false;
    }
    bool graph_is_model = true;
    if (P.has_graph) {
        if (gm != mm) graph_is_model = false;
        for (int64_t k = 0; k < gm && graph_is_model; ++k)
            if (gei[k] != mei[k] || gej[k] != mej[k] || (double)(-gew[k]) != mew[k])
                graph_is_model = false;
        for (int64_t k = 0; k < gm; ++k) P.total_w += gew[k];
    }
    const bool rule_is_psa = algo == 0 || (algo == 1 && alpha == 1) || (algo == 2 && p_stall == 0.0);
    // i < 2^30 and count < 2^30 let the packed kernel fold the first xorshift
    // of each absorb into per-trial constants (pbsa_device.cuh)
    const bool small_counters = n <= (1LL << 30) && cycles * t_res <= (1LL << 30);
    // time-averaged rule on the packed path: sum of alpha counts must stay < 64
    // (the history sum S of alpha counts of at most dmax < 2^L lives in L + 3 planes)
    int Lbits = 1;
    while ((1 << Lbits) - 1 < dmax) ++Lbits;
    const bool tapsa_packed = algo == 1 && alpha >= 2 && dmax <= 127 && alpha * dmax < (1LL << (Lbits + 3));
    // stalled rule on the packed path: per-p-bit threshold index into all cycles' tables
    const bool spsa_packed = algo == 2 && p_stall > 0.0 && cycles * (2 * dmax + 1) < (1LL << 31);
    // variability profile on the packed path: plain rule, finite lam/delta,
    // clamped periods below 256 (bit-sliced in at most 8 planes)
    const int64_t maxcount = cycles * t_res;
    // (PBSA_PACKED_VAR=0 sends variability runs to the active-list kernels)
    bool var_ok = (lam || native_prof) && !ideal && (algo == 0 || (algo == 2 && p_stall == 0.0));
    const char *venv = std::getenv("PBSA_PACKED_VAR");
    if (venv) var_ok = var_ok && venv[0] != '0';
    int64_t pmax = 0;
    bool var_uniform = true;
    if (var_ok && native_prof) {
        pmax = native_pmax;
        var_uniform = native_sig[2] == 0.0;
        var_ok = !native_overflow;
    } else if (var_ok) {
        for (int64_t k = 0; k < prow * n && var_ok; ++k) {
            var_ok = std::isfinite(lam[k]) && std::isfinite(delta[k]);
            const int64_t pc = std::min<int64_t>(period[k], maxcount);
            pmax = std::max(pmax, pc);
            var_uniform = var_uniform && period[k] == t_res;
        }
        var_ok = var_ok && pmax < 256;
    }
    const bool packed = (((rule_is_psa || tapsa_packed || spsa_packed) && ideal) || var_ok) && unit_J &&
                        zero_h && graph_is_model && dmax <= 127 && small_counters;
    if (native_prof && !(packed && var_ok))
        fail(PBSA_EINVAL, "native profiles run on the packed path only: a +-1 MAX-CUT model of degree "
                          "<= 127, the plain rule, and clamped periods below 256");
    if (rng_mode == PBSA_RNG_PHILOX && !packed)
        fail(PBSA_EINVAL, "rng_mode=philox runs on the packed path only: a +-1 MAX-CUT model of "
                          "degree <= 127 with pSA/TApSA/SpSA on an ideal profile, or the plain rule "
                          "with a variability profile");
    P.native = rng_mode == PBSA_RNG_PHILOX;
    P.nseed = rng_seed;
    P.first_trial = first_trial;
    P.var_mode = packed && var_ok;
    P.var_uniform = var_uniform;
    P.pmax = pmax;
    P.tapsa_packed = packed && tapsa_packed;
    P.spsa_packed = packed && spsa_packed && !rule_is_psa;
    P.tapsa_hist_from_raw = packed && algo == 1 && !P.tapsa_packed;
    P.path = packed ? PBSA_PATH_PACKED : PBSA_PATH_GENERAL;


    // per-trial key prefixes (streams.py: draws are absorb^3(key, tag, a, b))
    std::vector<uint64_t> kspin, kr, kst;
    host_trial_keys(keys, trials, P.Tp, kspin, kr, kst);
    P.kspin.upload(kspin, st);
    P.kr_host = kr;

    std::vector<uint32_t> rowptr(n + 1);
    for (int64_t i = 0; i <= n; ++i) rowptr[i] = (uint32_t)indptr[i];
    P.rowptr.upload(rowptr, st);

    if (packed) {
        // ---------------------------------------------------- packed setup
        P.dmax = (int)dmax;
        P.L = 1;
        while ((1 << P.L) - 1 < dmax) ++P.L;
        P.K = 2 * P.dmax + 1;
        std::vector<uint32_t> rowv, adjv;
        std::vector<uint16_t> adj16;
        host_csr(n, indptr, indices, values, rowv, adjv, adj16);
        // degree-4 regular graph (tori): rows at 4i, gathered with one 16-byte load
        P.reg4 = nnz == 4 * n;
        for (int64_t i = 0; i < n && P.reg4; ++i) P.reg4 = indptr[i] == 4 * i;
        if (const char *env = std::getenv("PBSA_REG4")) P.reg4 = P.reg4 && env[0] != '0';
        if (n <= 32768) P.adj16.upload(adj16, st); else P.adj.upload(adjv, st);
        std::vector<uint64_t> krg;
        std::vector<uint2> kfc;
        host_packed_consts(kr, krg, kfc);
        P.krg.upload(krg, st);
        P.kfc.upload(kfc, st);
        if (P.spsa_packed) {
            std::vector<uint64_t> kg(P.Tp);
            std::vector<uint2> kf(P.Tp);
            for (int64_t t = 0; t < P.Tp; ++t) {
                kg[t] = kst[t] + kGamma;
                const uint32_t lo = (uint32_t)kg[t], hi = (uint32_t)(kg[t] >> 32);
                const uint32_t Y = hi ^ (hi >> 30);
                kf[t] = make_uint2(lo ^ ((lo >> 30) | (hi << 2)), Y * 0x1CE4E5B9u);
            }
            P.kstg.upload(kg, st);
            P.kfs.upload(kf, st);
            // u = (H >> 11) 2^-53 < p  <=>  H < ceil(p 2^53) << 11   (p * 2^53 is exact)
            const double ps = std::ceil(std::ldexp(p_stall, 53));
            P.p_stall64 = ps >= 0x1p53 ? ~0ULL : ((uint64_t)ps << 11);
            // native: (X + 1/2) 2^-32 < p  <=>  X < S = ceil(p 2^32 - 1/2)   (exact in fp64)
            if (P.native) P.p_stall64 = (uint64_t)std::ceil(std::ldexp(p_stall, 32) - 0.5);
            P.sidx.alloc((size_t)P.W * 32 * n);
            if (const char *env = std::getenv("PBSA_SIDX_FULL")) P.sidx_full = env[0] != '0';
            P.i0_dev.upload(P.i0, st);
        }
        if (P.tapsa_packed) {
            // thresholds per (cycle, acc): acc = 2 S - f d in [-f dmax, f dmax],
            // f = min(c+1, alpha), entry acc + f dmax; inp = i0 * (acc / f) exactly as
            // _kernels.py:138 evaluates it
            P.K = (int)(2 * alpha * P.dmax + 1);
            std::vector<uint64_t> thr((size_t)cycles * P.K, ~0ULL);
            for (int64_t c = 0; c < cycles; ++c) {
                const int64_t f = std::min<int64_t>(c + 1, alpha);
                for (int64_t acc = -f * P.dmax; acc <= f * P.dmax; ++acc) {
                    const double t = pb_libm_tanh(P.i0[c] * ((double)acc / (double)f));
                    thr[(size_t)c * P.K + acc + f * P.dmax] = P.native ? threshold_native(t) : threshold_h64(t);
                }
            }
            P.thr.upload(thr, st);
            P.ring.alloc((size_t)P.W * alpha * P.L * n);
        } else {
            const std::vector<uint64_t> thr = host_plain_thresholds(P);
            P.thr.upload(thr, st);
            if (P.spsa_packed) {
                std::vector<uint32_t> hi(thr.size());
                for (size_t k = 0; k < thr.size(); ++k) hi[k] = (uint32_t)(thr[k] >> 32);
                P.thr_hi.upload(hi, st);
            }
        }
        for (auto &b : P.p_spins) b.alloc((size_t)P.W * n);
        P.pacc.alloc((size_t)(cycles + 1) * P.Tp);
        if (!P.var_mode) P.raw_last.alloc((size_t)n * P.Tp);

        // launch sequence: one sweep per cycle (counter c * t_res) ...
        if (!P.var_mode || P.var_uniform) {
            for (int64_t c = 0; c < cycles; ++c)
                P.plaunch.push_back({(uint32_t)(c * t_res), c, 1, 0, 0, true,
                                     c == cycles - 1});
        }
        if (P.var_mode)
            packed_variability_setup(P, n, trials, cycles, t_res, lam, delta, period, pstride, native_prof, st);
        P.plaunch.push_back({(uint32_t)(cycles * t_res), cycles, 1, 0, 0, false, false});

        packed_launch_shape(P, device, n, dmax);
        resident_setup(P, device, n, indptr, alpha, cycles, st);
        order_and_bucket_setup(P, n, indptr, st);
        P.updates_per_run = (int64_t)n * trials * cycles;
        if (P.var_mode && !P.var_uniform) {  // sum over p-bits of #{count < cycles t_res : period | count}
            int64_t ups = 0;
            for (uint8_t pc : P.pcl) ups += (maxcount + pc - 1) / pc;
            P.updates_per_run = ups;
        }
    } else {
        // --------------------------------------------------- general setup
        std::vector<uint32_t> colv(nnz);
        for (int64_t k = 0; k < nnz; ++k) colv[k] = (uint32_t)indices[k];
        P.col.upload(colv, st);
        P.val.upload(values, nnz, st);
        P.h.upload(hv, n, st);
        P.kr.upload(kr, st);
        P.kst.upload(kst, st);
        for (auto &b : P.g_spins) b.alloc((size_t)n * P.Tp);
        P.inputs.alloc((size_t)n * P.Tp);
        P.counts.alloc((size_t)n * P.Tp);
        if (algo == 1) P.hist.alloc((size_t)n * alpha * P.Tp);
        // profiles: [n] shared or [n][Tp] transposed from [T][n]
        std::vector<int64_t> distinct_periods;
        if (lam) {
            P.has_lam = P.has_delta = P.has_period = true;
            P.shared_profile = pstride == 0;
            const int64_t rows = P.shared_profile ? 1 : P.Tp;
            std::vector<double> l((size_t)n * rows, 1.0), d((size_t)n * rows, 0.0);
            std::vector<int32_t> p((size_t)n * rows, (int32_t)t_res);
            std::set<int64_t> ps;
            for (int64_t t = 0; t < (P.shared_profile ? 1 : trials); ++t)
                for (int64_t i = 0; i < n; ++i) {
                    const size_t src = (size_t)t * n + i;
                    const size_t dst = P.shared_profile ? (size_t)i : (size_t)i * P.Tp + t;
                    l[dst] = lam[src];
                    d[dst] = delta[src];
                    // periods beyond the last sub-step only ever fire at count 0
                    const int64_t pv = std::min<int64_t>(period[src], INT32_MAX);
                    p[dst] = (int32_t)pv;
                    ps.insert(pv);
                }
            P.lam.upload(l, st);
            P.delta.upload(d, st);
            P.period.upload(p, st);
            distinct_periods.assign(ps.begin(), ps.end());
        } else {
            distinct_periods.push_back(t_res);
        }
        // sub-steps where at least one p-bit of one trial fires
        for (int64_t c = 0; c < cycles; ++c)
            for (int64_t s = 0; s < t_res; ++s) {
                const int64_t count = c * t_res + s;
                for (int64_t pv : distinct_periods)
                    if (count % pv == 0) {
                        P.active_counts.push_back((uint32_t)count);
                        break;
                    }
            }
        // energy mode: exact integer accumulation when every term is integral
        double mag = 0.0;
        bool integral = true;
        for (int64_t k = 0; k < mm && integral; ++k) {
            integral = is_integral(mew[k]);
            mag += std::fabs(mew[k]);
        }
        for (int64_t i = 0; i < n && integral; ++i) {
            integral = is_integral(hv[i]);
            mag += std::fabs(hv[i]);
        }
        P.int_energy = integral && mag < 9.0e15;
        std::vector<uint32_t> a32(mm), b32(mm);
        for (int64_t k = 0; k < mm; ++k) {
            a32[k] = (uint32_t)mei[k];
            b32[k] = (uint32_t)mej[k];
        }
        P.me_i.upload(a32, st);
        P.me_j.upload(b32, st);
        if (P.int_energy) {
            // energy from per-edge disagreement counts: sum J s s = sum J - 2 sum_{differ} J;
            // for the MAX-CUT mapping (J = -w) the cut count alone gives it
            std::vector<int64_t> hi(n);
            std::vector<int32_t> wj(mm);
            bool any_h = false;
            for (int64_t k = 0; k < mm; ++k) {
                wj[k] = (int32_t)mew[k];
                P.sum_j += (int64_t)mew[k];
            }
            for (int64_t i = 0; i < n; ++i) {
                hi[i] = (int64_t)hv[i];
                any_h |= hi[i] != 0;
            }
            if (!(P.has_graph && graph_is_model)) {
                P.me_w32.upload(wj, st);
                P.dj_acc.alloc((size_t)cycles * P.Tp);
            }
            if (any_h) {
                P.h_int.upload(hi, st);
                P.e_acc.alloc((size_t)cycles * P.Tp);
            }
        } else {
            P.me_w.upload(mew, mm, st);
            P.e_f64.alloc((size_t)cycles * P.Tp);
        }
        std::vector<uint32_t> g32i(gm), g32j(gm);
        for (int64_t k = 0; k < gm; ++k) {
            g32i[k] = (uint32_t)gei[k];
            g32j[k] = (uint32_t)gej[k];
        }
        P.ge_i.upload(g32i, st);
        P.ge_j.upload(g32j, st);
        if (gm) P.ge_w.upload(gew, gm, st);
        if (gm && P.int_energy) {
            std::vector<int32_t> w32(gm);
            for (int64_t k = 0; k < gm; ++k) {
                if (gew[k] > INT32_MAX || gew[k] < INT32_MIN) fail(PBSA_EINVAL, "graph weight exceeds int32");
                w32[k] = (int32_t)gew[k];
            }
            P.ge_w32.upload(w32, st);
        }
        P.graph_is_model = P.has_graph && graph_is_model;
        P.cut_acc.alloc((size_t)cycles * P.Tp);
        // updates: sum over (trial, node) of ceil(cycles * t_res / period)
        const int64_t total = cycles * t_res;
        int64_t ups = 0;
        if (lam) {
            for (int64_t t = 0; t < trials; ++t)
                for (int64_t i = 0; i < n; ++i) {
                    const int64_t pv = period[(pstride ? t * n : 0) + i];
                    ups += (total + pv - 1) / pv;
                }
        } else {
            ups = trials * n * ((total + t_res - 1) / t_res);
        }
        P.updates_per_run = ups;
        if (P.int_energy)
            setup_active(P, n, indptr, indices, values, hv, lam, delta, period, pstride, trials,
                         cycles, t_res, algo, alpha, p_stall);
    }
    // mm/gm metadata for stats
    P.trace_cut.alloc((size_t)trials * cycles);
    P.trace_energy.alloc((size_t)trials * cycles);
    P.best.alloc((size_t)trials);
    CK(cudaStreamSynchronize(st));
    (void)mm;
}

}  // namespace pbsa_rt

// Host export of the launch-shape model (include/pbsa.h), for the CPU tests.
extern "C" int64_t pbsa_choose_phases_host(int64_t chunks, int64_t W, int64_t resident_warps, int64_t l2_budget,
                                           int *balance) {
    bool b = false;
    const int64_t pw = pbsa_rt::choose_phases(chunks, W, resident_warps, (size_t)std::max<int64_t>(0, l2_budget), &b);
    if (balance) *balance = b ? 1 : 0;
    return pw;
}
