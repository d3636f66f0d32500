// oneshot.cu -- one-shot batch calls (pbsa_anneal_loop_batch*), their plan cache and
// the device-list fan-out
#include "runtime.h"

namespace pbsa_rt {

// ------------------------------------------------------ one-shot plan cache
// A one-shot call of the plain rule with page-locked output buffers keeps its
// plan -- device buffers and the captured graph of the whole anneal with each
// word phase's output formatting and copies into the caller's buffers -- for
// the next call of the same shape.  Every call still uploads all of its
// inputs (CSR, per-trial keys and constants, threshold table) into the plan's
// buffers, replays the graph and writes all eight outputs; only buffer
// allocation and graph construction are amortised.  PBSA_PLAN_CACHE=0 turns
// it off; pbsa_plan_cache_clear() frees the cached plans.
struct CachedPlan {
    std::vector<uint64_t> key;
    pbsa_plan *P;
    uint64_t used;
};
std::mutex &plan_cache_mu() {
    static std::mutex *m = new std::mutex;  // (leaked: no destructor at exit)
    return *m;
}
std::vector<CachedPlan> &plan_cache() {
    static auto *v = new std::vector<CachedPlan>;
    return *v;
}
uint64_t g_cache_clock = 0;
constexpr size_t kPlanCacheCap = 2;

uint64_t hash_bytes(const void *p, size_t bytes, uint64_t h) {
    if (!p) return hmix64(h ^ 0x5bd1e995u);
    const uint8_t *b = static_cast<const uint8_t *>(p);
    size_t k = 0;
    for (; k + 8 <= bytes; k += 8) {
        uint64_t w;
        std::memcpy(&w, b + k, 8);
        h = (h ^ w) * 0x9E3779B97F4A7C15ULL;
        h ^= h >> 29;
    }
    uint64_t w = 0;
    std::memcpy(&w, b + k, bytes - k);
    return hmix64(h ^ w ^ (uint64_t)bytes);
}

bool pinned_or_null(const void *p) {
    if (!p) return true;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

pbsa_plan *plan_cache_take(const std::vector<uint64_t> &key) {
    std::lock_guard<std::mutex> lk(plan_cache_mu());
    auto &c = plan_cache();
    for (size_t k = 0; k < c.size(); ++k)
        if (c[k].key == key) {
            pbsa_plan *P = c[k].P;
            c.erase(c.begin() + k);
            return P;
        }
    return nullptr;
}

void plan_cache_put(std::vector<uint64_t> key, pbsa_plan *P) {
    std::vector<pbsa_plan *> evicted;
    {
        std::lock_guard<std::mutex> lk(plan_cache_mu());
        auto &c = plan_cache();
        for (const CachedPlan &e : c)
            if (e.key == key) {  // another thread's plan of this shape is cached already
                evicted.push_back(P);
                P = nullptr;
                break;
            }
        if (P) c.push_back({std::move(key), P, ++g_cache_clock});
        while (c.size() > kPlanCacheCap) {
            size_t old = 0;
            for (size_t k = 1; k < c.size(); ++k)
                if (c[k].used < c[old].used) old = k;
            evicted.push_back(c[old].P);
            c.erase(c.begin() + old);
        }
    }
    for (pbsa_plan *e : evicted) pbsa_plan_destroy(e);
}

// the outputs the graph writes, in PbsaHostOut order, with their byte sizes
void graph_outputs(const pbsa_plan &P, const PbsaHostOut &h, void *(&ptr)[5], size_t (&bytes)[5]) {
    const size_t T = (size_t)P.T, n = (size_t)P.n, C = (size_t)P.cycles;
    ptr[0] = h.spins;        bytes[0] = T * n;
    ptr[1] = h.inputs;       bytes[1] = T * n * 8;
    ptr[2] = h.trace_energy; bytes[2] = T * C * 8;
    ptr[3] = h.trace_cut;    bytes[3] = T * C * 8;
    ptr[4] = h.best;         bytes[4] = T * 8;
}

// Capture a cached one-shot plan's anneal with its phase outputs into one graph
// and index the graph's device-to-host copy nodes by output.
void capture_with_outputs(pbsa_plan &P, const PbsaHostOut &hout) {
    DeviceGuard dg(P.device);
    AllocStream as(P.stream);
    P.hout = hout;
    if (hout.spins) P.o_spins.alloc((size_t)P.T * P.n);
    if (hout.inputs) {
        P.o_raw16.alloc((size_t)P.T * P.n);
        CK(cudaMallocHost(reinterpret_cast<void **>(&P.h_raw), (size_t)P.T * P.n * sizeof(int16_t)));
    }
    CK(cudaStreamCreateWithFlags(&P.out_stream, cudaStreamNonBlocking));
    const int64_t nph = (P.W + P.phase_words - 1) / P.phase_words;
    P.cb_args.reserve(nph);  // (host nodes keep pointers into it)
    for (int64_t k = 0; k < nph; ++k) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        P.ev_phase.push_back(e);
    }
    cudaEvent_t ej;
    CK(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
    P.ev_phase.push_back(ej);  // (the join of the output stream; destroyed with the plan)
    CK(cudaStreamSynchronize(P.stream));  // buffers exist before the capture starts
    CK(cudaStreamBeginCapture(P.stream, cudaStreamCaptureModeThreadLocal));
    try {
        enqueue_run(P, P.mm_, P.gm_);
        CK(cudaEventRecord(ej, P.out_stream));
        CK(cudaStreamWaitEvent(P.stream, ej, 0));
    } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(P.stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    CK(cudaStreamEndCapture(P.stream, &P.graph));
    void *ptr[5];
    size_t bytes[5];
    graph_outputs(P, hout, ptr, bytes);
    size_t nn = 0;
    CK(cudaGraphGetNodes(P.graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(P.graph, nodes.data(), &nn));
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        CK(cudaGraphNodeGetType(nd, &ty));
        if (ty != cudaGraphNodeTypeMemcpy) continue;
        cudaMemcpy3DParms mp{};
        CK(cudaGraphMemcpyNodeGetParams(nd, &mp));
        const char *dst = static_cast<const char *>(mp.dstPtr.ptr);
        for (int k = 0; k < 5; ++k) {
            const char *b = static_cast<const char *>(ptr[k]);
            if (b && dst >= b && dst < b + bytes[k]) {
                P.out_nodes.push_back({nd, k});
                P.out_node_off.push_back((size_t)(dst - b));
                P.out_node_bytes.push_back(mp.extent.width * mp.extent.height * mp.extent.depth);
                P.out_node_src.push_back(mp.srcPtr.ptr);
                break;
            }
        }
    }
    for (int k = 0; k < 5; ++k) P.out_bound[k] = ptr[k];
    CK(cudaGraphInstantiate(&P.graph_exec, P.graph, 0));
}

// Point the graph's copy nodes at this call's output buffers.
void bind_outputs(pbsa_plan &P, const PbsaHostOut &hout) {
    void *ptr[5];
    size_t bytes[5];
    graph_outputs(P, hout, ptr, bytes);
    for (size_t j = 0; j < P.out_nodes.size(); ++j) {
        const int k = P.out_nodes[j].second;
        if (ptr[k] == P.out_bound[k]) continue;
        CK(cudaGraphExecMemcpyNodeSetParams1D(P.graph_exec, P.out_nodes[j].first,
                                              static_cast<char *>(ptr[k]) + P.out_node_off[j],
                                              P.out_node_src[j], P.out_node_bytes[j],
                                              cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < 5; ++k) P.out_bound[k] = ptr[k];
    P.hout = hout;
}

// This call's inputs into a cached plan's buffers (same sizes: the cache key
// fixes every shape), exactly as create_plan derives and uploads them.
void refresh_inputs(pbsa_plan &P, int64_t n, const int64_t *indptr, const int64_t *indices,
                    const double *values, const uint64_t *keys) {
    DeviceGuard dg(P.device);
    cudaStream_t st = P.stream;
    std::vector<uint64_t> kspin, kr, kst, krg;
    std::vector<uint2> kfc;
    host_trial_keys(keys, P.T, P.Tp, kspin, kr, kst);
    host_packed_consts(kr, krg, kfc);
    if (P.h_rowptr.empty()) {  // the model's CSR and the schedule's table (fixed by the key)
        host_csr(n, indptr, indices, values, P.h_rowptr, P.h_adj32, P.h_adj16);
        P.h_thr = host_plain_thresholds(P);
    }
    P.kspin.overwrite(kspin, st);
    P.krg.overwrite(krg, st);
    P.kfc.overwrite(kfc, st);
    P.rowptr.overwrite(P.h_rowptr, st);
    if (P.adj16.n) P.adj16.overwrite(P.h_adj16, st); else P.adj.overwrite(P.h_adj32, st);
    P.thr.overwrite(P.h_thr, st);
    P.kr_host = kr;
}

}  // namespace

extern "C" {

int pbsa_last_call_bytes(int64_t *h2d_bytes, int64_t *d2h_bytes) {
    if (h2d_bytes) *h2d_bytes = g_call_h2d;
    if (d2h_bytes) *d2h_bytes = g_call_d2h;
    return PBSA_OK;
}

int pbsa_plan_cache_clear(void) {
    std::vector<pbsa_plan *> all;
    {
        std::lock_guard<std::mutex> lk(plan_cache_mu());
        for (CachedPlan &e : plan_cache()) all.push_back(e.P);
        plan_cache().clear();
    }
    for (pbsa_plan *P : all) pbsa_plan_destroy(P);
    return PBSA_OK;
}

int pbsa_anneal_loop_batch_ex(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                              const double *values, const double *h, int64_t mm,
                              const int64_t *me_i, const int64_t *me_j, const double *me_w,
                              int64_t gm, const int64_t *ge_i, const int64_t *ge_j,
                              const int64_t *ge_w, const double *lam, const double *delta,
                              const int64_t *period, int64_t profile_stride, double i0_min,
                              double beta, int64_t cycles, int64_t t_res, int algo, int64_t alpha,
                              double p_stall, int64_t trials, const uint64_t *keys, int rng_mode,
                              uint64_t rng_seed, int64_t first_trial, int8_t *spins,
                              double *inputs, double *hist, int64_t *counts, double *trace_i0,
                              double *trace_energy, int64_t *trace_cut, int64_t *best_cut,
                              float *device_ms) {
    pbsa_plan *P = nullptr;
    const bool trace = std::getenv("PBSA_TRACE_CALL") != nullptr;  // (diagnostic timestamps)
    auto now_ms = [] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t_enter = now_ms();
    const char *cenv = std::getenv("PBSA_PLAN_CACHE");
    const bool cacheable = (!cenv || cenv[0] != '0') && lam == nullptr && indptr && n >= 1 && trials >= 1 &&
                           mm >= 0 && gm >= 0 && pinned_or_null(spins) && pinned_or_null(inputs) &&
                           pinned_or_null(trace_energy) && pinned_or_null(trace_cut) && pinned_or_null(best_cut);
    if (cacheable) {
        // the key: every scalar and the content of the model and graph (which
        // fix the path, launch structure and every value baked into the graph);
        // the per-trial keys are inputs uploaded on every call
        uint64_t hm = hash_bytes(indptr, (size_t)(n + 1) * 8, 1);
        const int64_t nnz = indptr[n];
        hm = hash_bytes(indices, (size_t)nnz * 8, hm);
        hm = hash_bytes(values, (size_t)nnz * 8, hm);
        hm = hash_bytes(h, (size_t)n * 8, hm);
        hm = hash_bytes(me_i, (size_t)mm * 8, hm);
        hm = hash_bytes(me_j, (size_t)mm * 8, hm);
        hm = hash_bytes(me_w, (size_t)mm * 8, hm);
        hm = hash_bytes(ge_i, (size_t)gm * 8, hm);
        hm = hash_bytes(ge_j, (size_t)gm * 8, hm);
        hm = hash_bytes(ge_w, (size_t)gm * 8, hm);
        uint64_t ps, i0b, bb;
        std::memcpy(&ps, &p_stall, 8);
        std::memcpy(&i0b, &i0_min, 8);
        std::memcpy(&bb, &beta, 8);
        const uint64_t outs = (spins ? 1 : 0) | (inputs ? 2 : 0) | (trace_energy ? 4 : 0) | (trace_cut ? 8 : 0) |
                              (best_cut ? 16 : 0);
        // (and the PBSA_* tuning variables, read at plan creation: a plan built
        // under other settings is another plan)
        for (char **e = environ; e && *e; ++e)
            if (std::strncmp(*e, "PBSA_", 5) == 0 && std::strncmp(*e, "PBSA_TRACE_CALL=", 16) != 0 &&
                std::strncmp(*e, "PBSA_DEVICES=", 13) != 0 && std::strncmp(*e, "PBSA_LIB=", 9) != 0)
                hm = hash_bytes(*e, std::strlen(*e), hm);
        std::vector<uint64_t> key = {(uint64_t)device, (uint64_t)n, (uint64_t)mm, (uint64_t)gm, (uint64_t)cycles,
                                     (uint64_t)t_res, (uint64_t)algo, (uint64_t)alpha, ps, (uint64_t)trials,
                                     (uint64_t)rng_mode, rng_seed, (uint64_t)first_trial, i0b, bb, outs, hm};
        const PbsaHostOut hout{spins, inputs, trace_energy, trace_cut, best_cut};
        P = plan_cache_take(key);
        int rc;
        if (P) {
            rc = guarded([&] {
                refresh_inputs(*P, n, indptr, indices, values, keys);
                bind_outputs(*P, hout);
            });
        } else {
            g_cached_oneshot = true;
            rc = pbsa_plan_create_ex(device, n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm,
                                     ge_i, ge_j, ge_w, lam, delta, period, profile_stride, i0_min,
                                     beta, cycles, t_res, algo, alpha, p_stall, trials, keys, rng_mode,
                                     rng_seed, first_trial, &P);
            g_cached_oneshot = false;
            if (rc != PBSA_OK) return rc;
            if (!P->capturing_outputs) {  // not the plain launched path: run it once, uncached
                rc = guarded([&] {
                    DeviceGuard dg(P->device);
                    CK(cudaEventRecord(P->ev_start, P->stream));
                    launch_run(*P);
                    CK(cudaEventRecord(P->ev_end, P->stream));
                    host_constant_outputs(P, hist, counts, trace_i0);
                    CK(cudaEventSynchronize(P->ev_end));
                    P->ran = true;
                    if (device_ms) CK(cudaEventElapsedTime(device_ms, P->ev_start, P->ev_end));
                    download_impl(P, spins, inputs, hist, counts, trace_i0, trace_energy, trace_cut,
                                  best_cut, true);
                });
                const std::string err = g_last_error;
                pbsa_plan_destroy(P);
                if (rc != PBSA_OK) g_last_error = err;
                return rc;
            }
            rc = guarded([&] { capture_with_outputs(*P, hout); });
        }
        if (rc == PBSA_OK)
            rc = guarded([&] {
                DeviceGuard dg(P->device);
                {
                    std::lock_guard<std::mutex> lk(P->cb_mu);
                    P->cb_done = 0;
                }
                const double t_ready = now_ms();
                CK(cudaEventRecord(P->ev_start, P->stream));
                CK(cudaGraphLaunch(P->graph_exec, P->stream));
                CK(cudaEventRecord(P->ev_end, P->stream));
                const double t_launched = now_ms();
                host_constant_outputs(P, hist, counts, trace_i0);  // host threads while the device runs
                const double t_host = now_ms();
                // fp64 inputs = i0_last * raw (_kernels.py:146) of each phase as it lands
                const double i0_last = P->i0[P->cycles - 1];
                for (size_t k = 0; inputs && k < P->phase_trials.size(); ++k) {
                    {
                        std::unique_lock<std::mutex> lk(P->cb_mu);
                        P->cb_cv.wait(lk, [&] { return P->cb_done > (int)k; });
                    }
                    const int64_t a0 = P->phase_trials[k].first * n, a1 = P->phase_trials[k].second * n;
                    const int16_t *src = P->h_raw;
                    parallel_for(a1 - a0, 1 << 18, [&](int64_t lo, int64_t hi) {
                        for (int64_t j = a0 + lo; j < a0 + hi; ++j) inputs[j] = i0_last * (double)src[j];
                    });
                }
                CK(cudaEventSynchronize(P->ev_end));
                P->ran = true;
                float dms = 0.f;
                CK(cudaEventElapsedTime(&dms, P->ev_start, P->ev_end));
                if (device_ms) *device_ms = dms;
                CK(cudaGetLastError());
                if (trace)
                    std::fprintf(stderr, "pbsa one-shot (cached plan): prepare %.2f ms, launch %.2f, host outputs %.2f, "
                                 "done at %.2f (device %.2f)\n", t_ready - t_enter, t_launched - t_ready,
                                 t_host - t_launched, now_ms() - t_enter, dms);
            });
        if (rc != PBSA_OK) {
            const std::string err = g_last_error;
            pbsa_plan_destroy(P);
            g_last_error = err;
            return rc;
        }
        {
            int64_t up = (int64_t)(P->kspin.bytes_up + P->krg.bytes_up + P->kfc.bytes_up + P->rowptr.bytes_up +
                                   P->adj16.bytes_up + P->adj.bytes_up + P->thr.bytes_up);
            int64_t down = 0;
            for (size_t j = 0; j < P->out_node_bytes.size(); ++j) down += (int64_t)P->out_node_bytes[j];
            if (inputs) down += P->T * P->n * (int64_t)sizeof(int16_t);
            g_call_h2d = up;
            g_call_d2h = down;
        }
        plan_cache_put(std::move(key), P);
        return PBSA_OK;
    }
    g_oneshot = true;
    int rc = pbsa_plan_create_ex(device, n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm,
                                 ge_i, ge_j, ge_w, lam, delta, period, profile_stride, i0_min,
                                 beta, cycles, t_res, algo, alpha, p_stall, trials, keys, rng_mode,
                                 rng_seed, first_trial, &P);
    g_oneshot = false;
    if (rc != PBSA_OK) return rc;
    if (P->pipelined) {
        // launch the phases directly; each phase's outputs stream back on
        // out_stream while the next anneals; the run-independent outputs are
        // written on the host meanwhile
        rc = guarded([&] {
            DeviceGuard dg(P->device);
            AllocStream as(P->stream);
            P->hout = PbsaHostOut{spins, inputs, trace_energy, trace_cut, best_cut};
            if (spins) P->o_spins.alloc((size_t)P->T * P->n);
            if (inputs) P->o_inputs.alloc((size_t)P->T * P->n);
            CK(cudaStreamCreateWithFlags(&P->out_stream, cudaStreamNonBlocking));
            const int64_t nph = (P->W + P->phase_words - 1) / P->phase_words;
            for (int64_t k = 0; k < nph; ++k) {
                cudaEvent_t e;
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                P->ev_phase.push_back(e);
            }
            const double t_created = now_ms();
            CK(cudaEventRecord(P->ev_start, P->stream));
            enqueue_run(*P, P->mm_, P->gm_);
            const double t_enqueued = now_ms();
            CK(cudaEventRecord(P->ev_end, P->stream));
            host_constant_outputs(P, hist, counts, trace_i0);
            const double t_host = now_ms();
            CK(cudaEventSynchronize(P->ev_end));
            const double t_dev = now_ms();
            P->ran = true;
            if (device_ms) CK(cudaEventElapsedTime(device_ms, P->ev_start, P->ev_end));
            CK(cudaStreamSynchronize(P->out_stream));
            CK(cudaGetLastError());
            if (trace) {
                float dms = 0.f;
                cudaEventElapsedTime(&dms, P->ev_start, P->ev_end);
                std::fprintf(stderr, "pbsa one-shot: create %.2f ms, enqueue %.2f, host outputs %.2f, "
                             "device done at %.2f (device %.2f), outputs done at %.2f\n",
                             t_created - t_enter, t_enqueued - t_created, t_host - t_enqueued,
                             t_dev - t_enter, dms, now_ms() - t_enter);
            }
        });
        const std::string err = g_last_error;
        const double t_d0 = now_ms();
        pbsa_plan_bytes(P, &g_call_h2d, &g_call_d2h);
        pbsa_plan_destroy(P);
        if (trace) std::fprintf(stderr, "pbsa one-shot: destroy %.2f ms, total %.2f ms\n", now_ms() - t_d0,
                                now_ms() - t_enter);
        if (rc != PBSA_OK) g_last_error = err;
        return rc;
    }
    // launch, write the run-independent outputs on the host while the device
    // anneals, then wait and download the rest
    rc = guarded([&] {
        DeviceGuard dg(P->device);
        CK(cudaEventRecord(P->ev_start, P->stream));
        launch_run(*P);
        CK(cudaEventRecord(P->ev_end, P->stream));
        host_constant_outputs(P, hist, counts, trace_i0);
        CK(cudaEventSynchronize(P->ev_end));
        P->ran = true;
        if (device_ms) CK(cudaEventElapsedTime(device_ms, P->ev_start, P->ev_end));
        download_impl(P, spins, inputs, hist, counts, trace_i0, trace_energy, trace_cut, best_cut,
                      true);
    });
    const std::string err = g_last_error;
    pbsa_plan_bytes(P, &g_call_h2d, &g_call_d2h);
    pbsa_plan_destroy(P);
    if (rc != PBSA_OK) g_last_error = err;
    return rc;
}

int pbsa_anneal_loop_batch_np(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                              const double *values, const double *h, int64_t mm, const int64_t *me_i,
                              const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                              const int64_t *ge_j, const int64_t *ge_w, const double *native_sigmas,
                              double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                              int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                              uint64_t rng_seed, int64_t first_trial, int8_t *spins, double *inputs,
                              double *hist, int64_t *counts, double *trace_i0, double *trace_energy,
                              int64_t *trace_cut, int64_t *best_cut, float *device_ms) {
    if (!native_sigmas) {
        g_last_error = "null native_sigmas";
        return PBSA_EINVAL;
    }
    if (native_sigmas[0] == 0.0 && native_sigmas[1] == 0.0 && native_sigmas[2] == 0.0)  // the ideal profile
        return pbsa_anneal_loop_batch_ex(device, n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm, ge_i,
                                         ge_j, ge_w, nullptr, nullptr, nullptr, 0, i0_min, beta, cycles, t_res,
                                         algo, alpha, p_stall, trials, keys, PBSA_RNG_PHILOX, rng_seed,
                                         first_trial, spins, inputs, hist, counts, trace_i0, trace_energy,
                                         trace_cut, best_cut, device_ms);
    pbsa_plan *P = nullptr;
    g_oneshot = true;
    int rc = pbsa_plan_create_np(device, n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm, ge_i,
                                 ge_j, ge_w, native_sigmas, i0_min, beta, cycles, t_res, algo, alpha,
                                 p_stall, trials, keys, rng_seed, first_trial, &P);
    g_oneshot = false;
    if (rc != PBSA_OK) return rc;
    rc = guarded([&] {
        DeviceGuard dg(P->device);
        CK(cudaEventRecord(P->ev_start, P->stream));
        launch_run(*P);
        CK(cudaEventRecord(P->ev_end, P->stream));
        host_constant_outputs(P, hist, counts, trace_i0);
        CK(cudaEventSynchronize(P->ev_end));
        P->ran = true;
        if (device_ms) CK(cudaEventElapsedTime(device_ms, P->ev_start, P->ev_end));
        download_impl(P, spins, inputs, hist, counts, trace_i0, trace_energy, trace_cut, best_cut, true);
    });
    const std::string err = g_last_error;
    pbsa_plan_bytes(P, &g_call_h2d, &g_call_d2h);
    pbsa_plan_destroy(P);
    if (rc != PBSA_OK) g_last_error = err;
    return rc;
}

int pbsa_native_profiles(int device, uint64_t rng_seed, int64_t first_trial, int64_t trials, int64_t n,
                         int64_t t_res, int64_t cycles, const double *native_sigmas, double *lam,
                         double *delta, int64_t *period) {
    return guarded([&] {
        if (!native_sigmas || !lam || !delta || !period) fail(PBSA_EINVAL, "null pointer");
        if (trials < 1 || n < 1 || t_res < 1 || cycles < 1) fail(PBSA_EINVAL, "sizes must be >= 1");
        DeviceGuard dg(device);
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        StreamHolder sh;
        sh.s = st;
        AllocStream as(st);
        const size_t cnt = (size_t)trials * n;
        DevBuf<double> l64, d64;
        DevBuf<uint8_t> pcl;
        DevBuf<int> ovf;
        l64.alloc(cnt);
        d64.alloc(cnt);
        pcl.alloc(cnt);
        ovf.alloc(1);
        CK(cudaMemsetAsync(ovf.p, 0, sizeof(int), st));
        pbsa::native_profiles<<<grid_for((int64_t)cnt, 256), 256, 0, st>>>(
            (uint32_t)rng_seed, (uint32_t)(rng_seed >> 32), (uint64_t)first_trial, trials, trials, (int)n,
            (int)t_res, native_sigmas[0], native_sigmas[1], native_sigmas[2], cycles * t_res, l64.p, d64.p,
            pcl.p, ovf.p);
        CK(cudaGetLastError());
        std::vector<uint8_t> pc(cnt);
        int ov = 0;
        CK(cudaMemcpyAsync(lam, l64.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(delta, d64.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(pc.data(), pcl.p, cnt, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&ov, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (ov) fail(PBSA_EINVAL, "a native period reaches 256 after clamping to cycles * t_res");
        for (size_t k = 0; k < cnt; ++k) period[k] = pc[k];
    });
}

int pbsa_anneal_loop_batch_devices(const int *devices, int ndev, int64_t n, const int64_t *indptr,
                                   const int64_t *indices, const double *values, const double *h,
                                   int64_t mm, const int64_t *me_i, const int64_t *me_j,
                                   const double *me_w, int64_t gm, const int64_t *ge_i,
                                   const int64_t *ge_j, const int64_t *ge_w, const double *lam,
                                   const double *delta, const int64_t *period,
                                   int64_t profile_stride, double i0_min, double beta,
                                   int64_t cycles, int64_t t_res, int algo, int64_t alpha,
                                   double p_stall, int64_t trials, const uint64_t *keys,
                                   int rng_mode, uint64_t rng_seed, int64_t first_trial,
                                   int8_t *spins, double *inputs, double *hist, int64_t *counts,
                                   double *trace_i0, double *trace_energy, int64_t *trace_cut,
                                   int64_t *best_cut, float *device_ms) {
    if (!devices || ndev < 1) {
        g_last_error = "need at least one device";
        return PBSA_EINVAL;
    }
    if (trials < 1) {
        g_last_error = "trials must be in [1, 2^24]";
        return PBSA_EINVAL;
    }
    // contiguous shards, interior edges at multiples of 4 (distributed.shard_range)
    std::vector<int64_t> edge(ndev + 1);
    for (int r = 0; r <= ndev; ++r)
        edge[r] = r == ndev ? trials : (trials * r / ndev) / 4 * 4;
    std::vector<int> rc(ndev, PBSA_OK);
    std::vector<float> ms(ndev, 0.f);
    std::vector<std::string> err(ndev);
    const int64_t a = std::max<int64_t>(alpha, 1);
    auto shard = [&](int r) {
        const int64_t lo = edge[r], hi = edge[r + 1], T = hi - lo;
        if (T <= 0) return;
        const size_t po = profile_stride ? (size_t)lo * (size_t)n : 0;
        rc[r] = pbsa_anneal_loop_batch_ex(
            devices[r], n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm, ge_i, ge_j, ge_w,
            lam ? lam + po : nullptr, delta ? delta + po : nullptr, period ? period + po : nullptr,
            profile_stride, i0_min, beta, cycles, t_res, algo, alpha, p_stall, T, keys + lo, rng_mode,
            rng_seed, first_trial + lo, spins ? spins + lo * n : nullptr, inputs ? inputs + lo * n : nullptr,
            hist ? hist + lo * n * a : nullptr, counts ? counts + lo * n : nullptr,
            trace_i0 ? trace_i0 + lo * cycles : nullptr, trace_energy ? trace_energy + lo * cycles : nullptr,
            trace_cut ? trace_cut + lo * cycles : nullptr, best_cut ? best_cut + lo : nullptr, &ms[r]);
        if (rc[r] != PBSA_OK) err[r] = g_last_error;  // (thread-local: copy it out)
    };
    std::vector<std::thread> pool;
    for (int r = 1; r < ndev; ++r) pool.emplace_back(shard, r);
    shard(0);
    for (auto &t : pool) t.join();
    float mx = 0.f;
    for (int r = 0; r < ndev; ++r) {
        if (rc[r] != PBSA_OK) {
            g_last_error = "shard " + std::to_string(r) + " (device " + std::to_string(devices[r]) + "): " + err[r];
            return rc[r];
        }
        mx = std::max(mx, ms[r]);
    }
    if (device_ms) *device_ms = mx;
    return PBSA_OK;
}

}  // extern "C"
