// launch.cu -- the anneal enqueue: one sweep launch per active sub-step, per-cycle
// statistics and trace finalisation, captured into a graph or launched directly
#include "runtime.h"

namespace pbsa_rt {

// The sweep-interval events are external event nodes inside a captured graph;
// a directly launched (pipelined) run records them normally.
cudaError_t record_sweep_event(const pbsa_plan &P, cudaEvent_t ev, cudaStream_t st) {
    return (P.pipelined || P.direct) && !P.capturing_outputs
               ? cudaEventRecord(ev, st)
               : cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
}

// Pipelined one-shot: once the words [w0, w1) have finished their last cut
// pass, format their trials' outputs (traces, spins, inputs) and copy them to
// the caller's host buffers on out_stream, while the main stream anneals the
// next phase.  Outputs of the plain rule on the packed path only.
// host node of a cached one-shot graph: phase k's int16 raw fields are in the
// staging buffer (runs on a driver thread: no CUDA calls, only a signal)
void CUDART_CB phase_landed(void *arg) {
    auto *cb = static_cast<pbsa_plan::PhaseCb *>(arg);
    {
        std::lock_guard<std::mutex> lk(cb->P->cb_mu);
        cb->P->cb_done = std::max(cb->P->cb_done, cb->k + 1);
    }
    cb->P->cb_cv.notify_all();
}

void enqueue_phase_outputs(pbsa_plan &P, int64_t w0, int64_t w1, int parity, int k) {
    const int TB = 256;
    cudaStream_t os = P.out_stream;
    CK(cudaEventRecord(P.ev_phase[k], P.stream));
    CK(cudaStreamWaitEvent(os, P.ev_phase[k], 0));
    const int64_t n = P.n, C = P.cycles;
    const int64_t t0 = w0 * 32, t1 = std::min<int64_t>(P.T, w1 * 32);
    if (t1 <= t0) return;
    const int64_t Tr = t1 - t0;
    pbsa::FinalArgs f{};
    f.pacc = P.pacc.p + t0;
    f.total_w = P.total_w;
    f.mode = 0;
    f.has_graph = P.has_graph;
    f.C = (int)C;
    f.Tp = (int)P.Tp;
    f.T = (int)Tr;
    f.trace_cut = P.trace_cut.p + t0 * C;
    f.trace_energy = P.trace_energy.p + t0 * C;
    f.best = P.best.p + t0;
    pbsa::finalize_traces<<<grid_for(Tr, TB), TB, 0, os>>>(f);
    ++P.launches;
    const PbsaHostOut &h = P.hout;
    if (h.trace_cut)
        CK(cudaMemcpyAsync(h.trace_cut + t0 * C, f.trace_cut, Tr * C * sizeof(int64_t), cudaMemcpyDeviceToHost, os));
    if (h.trace_energy)
        CK(cudaMemcpyAsync(h.trace_energy + t0 * C, f.trace_energy, Tr * C * sizeof(double),
                           cudaMemcpyDeviceToHost, os));
    if (h.best) CK(cudaMemcpyAsync(h.best + t0, f.best, Tr * sizeof(int64_t), cudaMemcpyDeviceToHost, os));
    if (h.spins) {
        pbsa::unpack_spins<<<grid_for(n * Tr, TB), TB, 0, os>>>(P.p_spins[parity].p + w0 * n, P.o_spins.p + t0 * n,
                                                                 (int)n, (int)(w1 - w0), (int)Tr);
        CK(cudaMemcpyAsync(h.spins + t0 * n, P.o_spins.p + t0 * n, Tr * n, cudaMemcpyDeviceToHost, os));
        ++P.launches;
    }
    if (h.inputs && P.capturing_outputs) {
        // int16 raw fields, trial-major, to the staging buffer; the host widens them
        dim3 tb(32, 8), g((unsigned)((Tr + 31) / 32), (unsigned)((n + 31) / 32));
        pbsa::transpose_tile<int16_t><<<g, tb, 0, os>>>(P.raw_last.p + t0, P.o_raw16.p + t0 * n, (int)n,
                                                         (int)P.Tp, (int)Tr);
        CK(cudaMemcpyAsync(P.h_raw + t0 * n, P.o_raw16.p + t0 * n, Tr * n * sizeof(int16_t),
                           cudaMemcpyDeviceToHost, os));
        P.phase_trials.push_back({t0, t1});
        P.cb_args.push_back({&P, (int)P.cb_args.size()});
        CK(cudaLaunchHostFunc(os, phase_landed, &P.cb_args.back()));
        ++P.launches;
    } else if (h.inputs) {
        pbsa::inputs_from_raw<<<grid_for(n * Tr, TB), TB, 0, os>>>(P.raw_last.p + t0, P.o_inputs.p + t0 * n,
                                                                   P.i0[C - 1], (int)n, (int)P.Tp, (int)Tr, 1.0);
        CK(cudaMemcpyAsync(h.inputs + t0 * n, P.o_inputs.p + t0 * n, Tr * n * sizeof(double),
                           cudaMemcpyDeviceToHost, os));
        ++P.launches;
    }
}

// One launch of the resident timing-spread cluster kernel for the whole run.
void enqueue_resident_timing(pbsa_plan &P) {
    cudaStream_t st = P.stream;

    pbsa::ResidentTimingArgs r{};
    r.s_in = P.p_spins[0].p;
    r.s_out = P.p_spins[1].p;
    r.rowptr = P.rowptr.p;
    r.adj16 = P.adj16.p;
    r.kfc = P.kfc.p;
    r.krg = P.krg.p;
    r.prof = P.prof16.p;
    r.lam64 = P.lam64.p;
    r.del64 = P.del64.p;
    r.pplanes = P.pplanes.p;
    r.divs = P.vdivs.p;
    r.launches = P.rlaunch.p;
    r.nlaunch = (int)P.rlaunch.n;
    r.i0 = P.i0_dev.p;
    r.pacc = P.pacc.p;
    r.inp_out = P.inp_var.p;
    r.n = (int)P.n;
    r.W = (int)P.W;
    r.Tp = (int)P.Tp;
    r.nplanes = P.nplanes;
    r.cycles = (int)P.cycles;
    r.margin = P.var_margin;
    r.prof_smem = P.res_prof_smem ? 1 : 0;
    r.split = P.res_split ? 1 : 0;
    if (P.native) {
        pbsa::philox_round_keys((uint32_t)P.nseed, (uint32_t)(P.nseed >> 32), r.rk);
        r.ngroup = (uint32_t)(P.first_trial / 4);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(P.W * P.res_cs));
    cfg.blockDim = dim3((unsigned)P.res_threads);
    cfg.dynamicSmemBytes = P.res_smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)P.res_cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, resident_timing_for(P.L, P.native), r));
    ++P.launches;
    P.sweep_launches = (int64_t)P.rlaunch.n - 1;
}

// One launch of the resident cluster kernel for the whole run (plain rule,
// varied profile without timing spread, TApSA).
void enqueue_resident(pbsa_plan &P) {
    cudaStream_t st = P.stream;
    const int TB = 256;

    if (P.use_cache) {
        pbsa::packed_cache_init<<<grid_for(P.W * P.chunks * 1024, TB), TB, 0, st>>>(
            P.acache.p, P.krg.p, (int)P.n, P.chunks, (int)P.W, nullptr);
        ++P.launches;
    }
    pbsa::ResidentArgs r{};
    r.s_in = P.p_spins[0].p;
    r.s_out = P.p_spins[1].p;
    r.rowptr = P.rowptr.p;
    r.adj16 = P.adj16.p;
    r.kfc = P.kfc.p;
    r.acache = P.use_cache ? P.acache.p : nullptr;
    r.krg = P.krg.p;
    r.thr = P.thr.p;
    r.pacc = P.pacc.p;
    r.raw_out = P.raw_last.p;
    r.n = (int)P.n;
    r.W = (int)P.W;
    r.Tp = (int)P.Tp;
    r.K = P.K;
    r.dmax = P.dmax;
    r.chunks = P.chunks;
    r.cycles = (int)P.cycles;
    r.t_res = (int)P.t_res;
    if (P.var_mode) {
        r.prof = P.prof.p;
        r.lam64 = P.lam64.p;
        r.del64 = P.del64.p;
        r.i0 = P.i0_dev.p;
        r.inp_out = P.inp_var.p;
        r.margin = P.var_margin;
    }
    if (P.native) {
        pbsa::philox_round_keys((uint32_t)P.nseed, (uint32_t)(P.nseed >> 32), r.rk);
        r.ngroup = (uint32_t)(P.first_trial / 4);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(P.W * P.res_cs));
    cfg.blockDim = dim3((unsigned)P.res_threads);
    cfg.dynamicSmemBytes = P.res_smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)P.res_cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (P.res_tapsa) {
        r.ring = P.ring.p;
        r.alpha = (int)P.alpha;
    }
    CK(cudaLaunchKernelEx(&cfg, resident_kernel_for(P.L, P.use_cache, P.var_mode, P.native, P.res_tapsa), r));
    ++P.launches;
    P.sweep_launches = P.cycles;
}

// The launched packed sweeps.  Word phases run one after another so that a
// phase's first-absorb cache (PW words x n x 256 B) stays L2-resident across
// its cycles; inside a phase, independent word groups run as concurrent
// chains (graph branches) so one chain's launch gaps and tail are filled by
// the others' blocks.  Returns the spin buffer holding the final state.
int enqueue_packed_phases(pbsa_plan &P, PackedKernel kern_up, PackedKernel kern_cut, size_t smem) {
    cudaStream_t st = P.stream;
    const int TB = 256;
    const int G = (int)P.chain_streams.size() + 1;
    int cur = 0;
    for (int64_t p0 = 0; p0 < P.W; p0 += P.phase_words) {
        const int64_t p1 = std::min<int64_t>(P.W, p0 + P.phase_words);
        if (P.use_cache) {
            pbsa::packed_cache_init<<<grid_for((p1 - p0) * P.chunks * 1024, TB), TB, 0, st>>>(
                P.acache.p, P.krg.p + p0 * 32, (int)P.n, P.chunks, (int)(p1 - p0),
                P.order.n ? P.order.p : nullptr);
            ++P.launches;
        }
        if (G > 1) {
            CK(cudaEventRecord(P.ev_fork, st));
            for (cudaStream_t cs : P.chain_streams) CK(cudaStreamWaitEvent(cs, P.ev_fork, 0));
        }
        const int64_t per = (p1 - p0 + G - 1) / G;
        // launches interleaved across the chains (round robin), so a directly
        // launched run fills every chain's queue evenly; a captured graph is
        // the same either way (each chain keeps its own order)
        std::vector<int> cur_g(G, 0);
        for (const pbsa_plan::PLaunch &pl : P.plaunch) {
            for (int g = 0; g < G; ++g) {
                const int64_t w0 = p0 + g * per, w1 = std::min<int64_t>(p1, w0 + per);
                if (w0 >= w1) continue;
                cudaStream_t cs = g == 0 ? st : P.chain_streams[g - 1];
                const int blocks = (int)grid_for((w1 - w0) * P.warps_per_word, pbsa::kPackedWarps);
                int &cur = cur_g[g];
                    const int64_t c = pl.cycle;
                    pbsa::PackedArgs a{};
                    a.sold = P.p_spins[cur].p + w0 * P.n;
                    a.snew = P.p_spins[cur ^ 1].p + w0 * P.n;
                    a.rowptr = P.rowptr.p;
                    a.adj = P.adj.n ? P.adj.p : nullptr;
                    a.adj16 = P.adj16.n ? P.adj16.p : nullptr;
                    a.order = P.order.n ? P.order.p : nullptr;
                    a.krg = P.krg.p + w0 * 32;
                    a.kfc = P.kfc.p + w0 * 32;
                    a.acache = P.use_cache ? P.acache.p + (size_t)(w0 - p0) * P.chunks * 1024 : nullptr;
                    const int64_t cc = std::min<int64_t>(c, P.cycles - 1);
                    a.thr = P.thr.p + (size_t)cc * P.K;
                    a.pacc = P.pacc.p + (size_t)c * P.Tp + w0 * 32;
                    a.raw_out = (c == P.cycles - 1 && !P.var_mode) ? P.raw_last.p + w0 * 32 : nullptr;
                    a.n = (int)P.n;
                    a.W = (int)(w1 - w0);
                    a.Tp = (int)P.Tp;
                    a.K = P.K;
                    a.dmax = P.dmax;
                    a.warps_per_word = P.warps_per_word;
                    a.cta_flush = (P.cta_flush && P.warps_per_word % pbsa::kPackedWarps == 0) ? 1 : 0;
                // (L1 prefetch of the hash-cache tiles: off since the instruction trims
                // of late round 2 -- C4 9.25e11 with it, 9.47e11 without; the loads hit
                // L1 3 % of the time either way.  PBSA_CACHE_PREFETCH=1 enables it)
                a.cache_prefetch = 0;
                // (the bucket kernel keeps the 1-D grid: G55 C3 measured 7 % slower 2-D)
                a.grid2d = a.cta_flush && !(P.bucket && pl.update);
                if (const char *env = std::getenv("PBSA_GRID2D")) a.grid2d = a.cta_flush && env[0] == '1';
                if (const char *env = std::getenv("PBSA_CACHE_PREFETCH")) a.cache_prefetch = env[0] == '1';
                    a.chunks = P.chunks;
                    a.count = pl.count;
                    a.do_update = pl.update;
                    a.reg4 = P.reg4 ? 1 : 0;
                    if (P.native) {
                        a.nk0 = (uint32_t)P.nseed;
                        a.nk1 = (uint32_t)(P.nseed >> 32);
                        a.ngroup = (uint32_t)((P.first_trial + w0 * 32) / 4);
                        pbsa::philox_round_keys(a.nk0, a.nk1, a.rk);
                    }
                    a.do_cut = pl.do_cut;
                    if (P.var_mode) {
                        const size_t off = (size_t)w0 * 32 * P.n;
                        a.prof = P.var_uniform ? P.prof.p + off : nullptr;
                        a.prof16 = P.var_uniform ? nullptr : P.prof16.p + off;
                        a.lam64 = P.lam64.p + off;
                        a.del64 = P.del64.p + off;
                        a.pplanes = P.var_uniform ? nullptr : P.pplanes.p + (size_t)w0 * P.nplanes * P.n;
                        a.divs = P.var_uniform ? nullptr : (P.bucket ? P.bdivs.p : P.vdivs.p) + pl.div_off;
                        if (P.bucket) {
                            const size_t toff = (size_t)w0 * P.chunks;
                            a.brec = P.brec.p + toff * 1024;
                            a.boff = P.boff.p + toff * (P.nclass + 1);
                            a.nclass = P.nclass;
                            a.cper = P.bcper.p;
                            a.maxcount = (uint32_t)(P.cycles * P.t_res);
                        }
                        a.ndiv = pl.ndiv;
                        a.nplanes = P.nplanes;
                        a.i0 = P.i0[cc];
                        a.i0f = (float)P.i0[cc];
                        a.margin = P.var_margin;
                        a.inp_out = pl.inp ? P.inp_var.p + off : nullptr;
                    }
                    if (P.spsa_packed) {
                        a.sidx = P.sidx.p + (size_t)w0 * 32 * P.n;
                        a.thr_hi_all = P.thr_hi.p;
                        a.kfs = P.kfs.p + w0 * 32;
                        a.kst = P.kstg.p + w0 * 32;
                        a.thr_all = P.thr.p;
                        a.p_stall64 = P.p_stall64;
                        a.cycle = (int)cc;
                        a.Kc = P.K;
                        a.sidx_full = P.sidx_full ? 1 : 0;
                    }
                    if (P.tapsa_packed) {
                        a.ring = P.ring.p + (size_t)w0 * P.alpha * P.L * P.n;
                        a.alpha = (int)P.alpha;
                        a.slot = (int)(cc % P.alpha);
                        a.filled = (int)std::min<int64_t>(cc + 1, P.alpha);
                    }
                    {
                        // programmatic dependent launch: the next sub-step's prologue
                        // overlaps this one's tail (the kernel waits on griddepcontrol)
                        cudaLaunchConfig_t cfg{};
                        // one word per block: a 2-D grid (blocks of a word, words)
                        cfg.gridDim = a.grid2d ? dim3((unsigned)(P.warps_per_word / pbsa::kPackedWarps),
                                                         (unsigned)(w1 - w0))
                                                  : dim3((unsigned)blocks);
                        cfg.blockDim = dim3(pbsa::kPackedThreads);
                        cfg.dynamicSmemBytes = (pl.update && P.var_mode && !P.var_uniform)
                                                   ? (P.bucket ? pbsa::bucket_smem_bytes(P.L) : pbsa::kTimingSmem)
                                                   : smem;
                        cfg.stream = cs;
                        cudaLaunchAttribute attr[1];
                        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                        attr[0].val.programmaticStreamSerializationAllowed = P.use_pdl ? 1 : 0;
                        cfg.attrs = attr;
                        cfg.numAttrs = 1;
                        CK(cudaLaunchKernelEx(&cfg, pl.update ? kern_up : kern_cut, a));
                    }
                    CK(cudaGetLastError());
                    ++P.launches;
                    if (pl.update) {
                        if (g == 0 && p0 == 0) ++P.sweep_launches;
                        cur ^= 1;
                    }
            }
        }
        for (int g = 1; g < G; ++g) {
            const int64_t w0 = p0 + g * per;
            if (w0 >= std::min<int64_t>(p1, w0 + per)) continue;
            CK(cudaEventRecord(P.ev_join[g - 1], P.chain_streams[g - 1]));
            CK(cudaStreamWaitEvent(st, P.ev_join[g - 1], 0));
        }
        cur = cur_g[0];
        if (P.pipelined) enqueue_phase_outputs(P, p0, p1, cur, (int)(p0 / P.phase_words));
    }
    return cur;
}

// The general (int8, trial-major) path: one substep or active-list launch
// per active sub-step, per-cycle statistics, trace finalisation.
void enqueue_general(pbsa_plan &P, int64_t mm, int64_t gm) {
    cudaStream_t st = P.stream;
    const int TB = 256;

    pbsa::init_general<<<grid_for(P.n * P.Tp, TB), TB, 0, st>>>(P.g_spins[0].p, P.kspin.p,
                                                                (int)P.n, (int)P.Tp);
    if (P.inputs.n) CK(cudaMemsetAsync(P.inputs.p, 0, P.inputs.n * sizeof(double), st));
    if (P.counts.n) CK(cudaMemsetAsync(P.counts.p, 0, P.counts.n * sizeof(int32_t), st));
    if (P.a_inputs.n) CK(cudaMemsetAsync(P.a_inputs.p, 0, P.a_inputs.n * sizeof(double), st));
    if (P.a_counts.n) CK(cudaMemsetAsync(P.a_counts.p, 0, P.a_counts.n * sizeof(int32_t), st));
    if (P.nflips.n) CK(cudaMemsetAsync(P.nflips.p, 0, P.nflips.n * sizeof(uint32_t), st));
    if (P.hist.n) CK(cudaMemsetAsync(P.hist.p, 0, P.hist.n * sizeof(double), st));
    if (P.hist_i.n) CK(cudaMemsetAsync(P.hist_i.p, 0, P.hist_i.n * sizeof(int32_t), st));
    CK(cudaMemsetAsync(P.cut_acc.p, 0, P.cut_acc.n * sizeof(unsigned long long), st));
    if (P.e_acc.n) CK(cudaMemsetAsync(P.e_acc.p, 0, P.e_acc.n * sizeof(unsigned long long), st));
    if (P.dj_acc.n) CK(cudaMemsetAsync(P.dj_acc.p, 0, P.dj_acc.n * sizeof(unsigned long long), st));
    P.launches += 1;
    CK(record_sweep_event(P, P.ev_sweep0, st));
    int cur = 0;
    size_t ai = 0, li = 0;
    const int sm_chunks = std::max<int64_t>(1, std::min<int64_t>(64, (std::max(mm, gm) + 255) / 256));
    for (int64_t c = 0; c < P.cycles; ++c) {
        // active-list mode: in-place spins, staged + scattered per sub-step
        while (P.active_mode && li < P.alaunch.size() && P.alaunch[li].cycle == c) {
            const pbsa_plan::ALaunch &L = P.alaunch[li];
            pbsa::ActiveArgs a{};
            a.s = P.g_spins[0].p;
            a.st_g = P.st_g.p;
            a.st_v = P.st_v.p;
            a.list = P.alist.p;
            a.desc = P.adesc.p + L.desc_off;
            a.ndesc = L.ndesc;
            a.total = L.total;
            a.rowptr = P.rowptr.p;
            a.col = P.col.p;
            a.vali = P.vali.p;
            a.hi = P.hi32.n ? P.hi32.p : nullptr;
            a.lam = P.has_lam ? P.lam.p : nullptr;
            a.delta = P.has_delta ? P.delta.p : nullptr;
            a.shared_profile = P.shared_profile;
            a.inputs = P.a_inputs.p;
            a.counts = P.a_counts.p;
            a.hist = P.hist_i.p;
            a.Np = (int64_t)P.alist.n;
            a.kr = P.kr.p;
            a.kst = P.kst.p;
            a.thr = P.athr.n ? P.athr.p + (size_t)c * P.Kt : nullptr;
            a.rawmin = P.rawmin;
            a.tshift = P.tshift;
            a.tmask = P.tmask;
            a.Tp = (int)P.Tp;
            a.alpha = (int)P.alpha;
            a.algo = P.algo;
            a.i0 = P.i0[c];
            a.p_stall = P.p_stall;
            a.count = L.count;
            if (P.fast) {
                pbsa::FastArgs f{};
                f.s = P.g_spins[0].p;
                f.list = P.alist.p;
                f.desc = a.desc;
                f.ndesc = L.ndesc;
                f.total = L.total;
                f.rowptr = P.rowptr.p;
                f.col = P.col.p;
                f.vali = P.vali.p;
                f.hi = a.hi;
                f.prof = P.aprof.n ? P.aprof.p : nullptr;
                f.lam64 = P.lam.p;
                f.del64 = P.delta.p;
                f.shared_profile = P.shared_profile;
                f.thr = a.thr;
                f.rawmin = P.rawmin;
                f.kfc = P.kfc.p;
                f.krg = P.krg.p;
                f.tshift = P.tshift;
                f.tmask = P.tmask;
                f.Tp = (int)P.Tp;
                f.count = L.count;
                f.i0 = P.i0[c];
                f.i0f = (float)P.i0[c];
                f.margin = P.var_margin;
                f.inputs = (int64_t)L.count >= P.cycles * P.t_res - P.apmax ? P.a_inputs.p : nullptr;
                f.flips = P.flips.p;
                f.nflips = P.nflips.p + li;
                pbsa::active_fast<<<grid_for(L.total, TB), TB, 0, st>>>(f);
                CK(cudaGetLastError());
                pbsa::apply_flips<<<grid_for(L.total, TB), TB, 0, st>>>(P.g_spins[0].p, P.flips.p,
                                                                       P.nflips.p + li);
            } else {
                pbsa::general_active<<<grid_for(L.total, TB), TB, 0, st>>>(a);
                CK(cudaGetLastError());
                pbsa::general_scatter<<<grid_for(L.total, TB), TB, 0, st>>>(P.g_spins[0].p, P.st_g.p,
                                                                           P.st_v.p, L.total);
            }
            P.launches += 2;
            ++P.sweep_launches;
            ++li;
        }
        while (!P.active_mode && ai < P.active_counts.size() && P.active_counts[ai] < (uint64_t)(c + 1) * P.t_res) {
            pbsa::GeneralArgs a{};
            a.sold = P.g_spins[cur].p;
            a.snew = P.g_spins[cur ^ 1].p;
            a.rowptr = P.rowptr.p;
            a.col = P.col.p;
            a.val = P.val.p;
            a.h = P.h.p;
            a.lam = P.has_lam ? P.lam.p : nullptr;
            a.delta = P.has_delta ? P.delta.p : nullptr;
            a.period = P.has_period ? P.period.p : nullptr;
            a.shared_profile = P.shared_profile;
            a.inputs = P.inputs.p;
            a.counts = P.counts.p;
            a.hist = P.hist.p;
            a.kr = P.kr.p;
            a.kst = P.kst.p;
            a.n = (int)P.n;
            a.Tp = (int)P.Tp;
            a.T = (int)P.T;
            a.algo = P.algo;
            a.alpha = (int)P.alpha;
            a.t_res = (int)P.t_res;
            a.i0 = P.i0[c];
            a.p_stall = P.p_stall;
            a.count = P.active_counts[ai];
            pbsa::general_substep<<<grid_for(P.n * P.Tp, TB), TB, 0, st>>>(a);
            CK(cudaGetLastError());
            ++P.launches;
            ++P.sweep_launches;
            cur ^= 1;
            ++ai;
        }
        if (P.int_energy) {
            const int64_t mx = std::max(gm, P.graph_is_model ? (int64_t)0 : mm);
            const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(256, mx / 256));
            dim3 grid(chunks, (unsigned)grid_for(P.Tp / 4, TB));
            if (gm) {
                pbsa::differ_count<<<grid, TB, 0, st>>>(P.g_spins[cur].p, P.ge_i.p, P.ge_j.p,
                                                        P.ge_w32.p, gm, (int)(P.Tp / 4), chunks,
                                                        P.cut_acc.p + (size_t)c * P.Tp);
                ++P.launches;
            }
            if (!P.graph_is_model && mm) {
                pbsa::differ_count<<<grid, TB, 0, st>>>(P.g_spins[cur].p, P.me_i.p, P.me_j.p,
                                                        P.me_w32.p, mm, (int)(P.Tp / 4), chunks,
                                                        P.dj_acc.p + (size_t)c * P.Tp);
                ++P.launches;
            }
            if (P.e_acc.n) {  // sum_i h_i s_i
                pbsa::StatsArgs s{};
                s.s = P.g_spins[cur].p;
                s.hi = P.h_int.p;
                s.n = (int)P.n;
                s.Tp = (int)P.Tp;
                s.T = (int)P.T;
                s.chunks = sm_chunks;
                s.cut_acc = P.cut_acc.p + (size_t)c * P.Tp;
                s.e_acc = P.e_acc.p + (size_t)c * P.Tp;
                dim3 g2(sm_chunks, (unsigned)grid_for(P.T, TB));
                pbsa::general_stats<<<g2, TB, 0, st>>>(s);
                ++P.launches;
            }
        } else {
            pbsa::StatsArgs s{};
            s.s = P.g_spins[cur].p;
            s.ge_i = P.ge_i.p;
            s.ge_j = P.ge_j.p;
            s.ge_w = P.ge_w.p;
            s.gm = gm;
            s.n = (int)P.n;
            s.Tp = (int)P.Tp;
            s.T = (int)P.T;
            s.chunks = sm_chunks;
            s.cut_acc = P.cut_acc.p + (size_t)c * P.Tp;
            dim3 grid(sm_chunks, (unsigned)grid_for(P.T, TB));
            pbsa::general_stats<<<grid, TB, 0, st>>>(s);
            ++P.launches;
        }
        if (!P.int_energy) {
            pbsa::general_energy_f64<<<grid_for(P.T, 128), 128, 0, st>>>(
                P.g_spins[cur].p, P.h.p, P.me_i.p, P.me_j.p, P.me_w.p, mm, (int)P.n,
                (int)P.Tp, (int)P.T, P.e_f64.p + (size_t)c * P.Tp);
            ++P.launches;
        }
    }
    CK(record_sweep_event(P, P.ev_sweep1, st));
    P.final_parity = cur;
    pbsa::FinalArgs f{};
    f.cut_acc = P.cut_acc.p;
    f.e_acc = P.e_acc.n ? P.e_acc.p : nullptr;
    f.dj_acc = P.dj_acc.p;
    f.sum_j = P.sum_j;
    f.graph_is_model = P.graph_is_model;
    f.e_f64 = P.e_f64.p;
    f.mode = P.int_energy ? 1 : 2;
    f.has_graph = P.has_graph;
    f.C = (int)P.cycles;
    f.Tp = (int)P.Tp;
    f.T = (int)P.T;
    f.trace_cut = P.trace_cut.p;
    f.trace_energy = P.trace_energy.p;
    f.best = P.best.p;
    pbsa::finalize_traces<<<grid_for(P.T, TB), TB, 0, st>>>(f);
    ++P.launches;
}

void enqueue_run(pbsa_plan &P, int64_t mm, int64_t gm) {
    cudaStream_t st = P.stream;
    const int TB = 256;
    P.launches = 0;
    P.sweep_launches = 0;
    if (P.path == PBSA_PATH_PACKED) {
        pbsa::init_packed<<<grid_for(P.n * P.W, TB), TB, 0, st>>>(P.p_spins[0].p, P.kspin.p,
                                                                   (int)P.n, (int)P.W);
        CK(cudaMemsetAsync(P.pacc.p, 0, P.pacc.n * sizeof(unsigned long long), st));
        P.launches += 1;
        PackedKernel kern_up = P.bucket ? bucket_kernel_for(P.L, P.native)
                                        : packed_kernel_for(P.L, true, P.use_cache, P.tapsa_packed, P.spsa_packed,
                                                            P.var_mode ? (P.var_uniform ? 1 : 2) : 0, P.native);
        PackedKernel kern_cut = packed_kernel_for(P.L, false, false);
        const size_t smem = (size_t)std::max(P.K, (P.dmax + 1) * 32) * 8 + 512 + 2 * pbsa::kPackedWarps * 32 * 8 + 16 +
                             pbsa::kPackedFlushBytes;
        CK(record_sweep_event(P, P.ev_sweep0, st));
        int cur = 1;  // (the spin buffer holding the final state)
        if (P.resident && P.res_timing)
            enqueue_resident_timing(P);
        else if (P.resident)
            enqueue_resident(P);
        else
            cur = enqueue_packed_phases(P, kern_up, kern_cut, smem);
        CK(record_sweep_event(P, P.ev_sweep1, st));
        P.final_parity = cur;
        if (!P.pipelined) {
            pbsa::FinalArgs f{};
            f.pacc = P.pacc.p;
            f.total_w = P.total_w;
            f.mode = 0;
            f.has_graph = P.has_graph;
            f.C = (int)P.cycles;
            f.Tp = (int)P.Tp;
            f.T = (int)P.T;
            f.trace_cut = P.trace_cut.p;
            f.trace_energy = P.trace_energy.p;
            f.best = P.best.p;
            pbsa::finalize_traces<<<grid_for(P.T, TB), TB, 0, st>>>(f);
            ++P.launches;
        }
    } else {
        enqueue_general(P, mm, gm);
    }
    CK(cudaGetLastError());
}

void host_constant_outputs(pbsa_plan *P, double *hist, int64_t *counts, double *trace_i0);
// The whole anneal on the plan stream: the captured graph, or (one-shot
// plans) the launches themselves.
void launch_run(pbsa_plan &P) {
    if (P.direct) {
        enqueue_run(P, P.mm_, P.gm_);
        CK(cudaGetLastError());
    } else {
        CK(cudaGraphLaunch(P.graph_exec, P.stream));
    }
}
void download_impl(pbsa_plan *P, int8_t *spins, double *inputs, double *hist, int64_t *counts,
                   double *trace_i0, double *trace_energy, int64_t *trace_cut, int64_t *best_cut,
                   bool consts_done);

}  // namespace pbsa_rt
