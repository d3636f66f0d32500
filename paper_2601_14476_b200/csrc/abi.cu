// abi.cu -- the plan entry points of include/pbsa.h and the output download
#include "runtime.h"


// =================================================================== C ABI
extern "C" {

int pbsa_abi_version(void) { return PBSA_ABI_VERSION; }

const char *pbsa_last_error(void) { return g_last_error.c_str(); }

int pbsa_device_count(int *count) {
    return guarded([&] {
        if (!count) fail(PBSA_EINVAL, "null count");
        CK(cudaGetDeviceCount(count));
    });
}

int pbsa_plan_create(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                     const double *values, const double *h, int64_t mm, const int64_t *me_i,
                     const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                     const int64_t *ge_j, const int64_t *ge_w, const double *lam,
                     const double *delta, const int64_t *period, int64_t profile_stride,
                     double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                     int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                     pbsa_plan **out) {
    return pbsa_plan_create_ex(device, n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm,
                               ge_i, ge_j, ge_w, lam, delta, period, profile_stride, i0_min, beta,
                               cycles, t_res, algo, alpha, p_stall, trials, keys, PBSA_RNG_REPLAY,
                               0, 0, out);
}

}  // extern "C"

namespace pbsa_rt {
int plan_create_impl(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                     const double *values, const double *h, int64_t mm, const int64_t *me_i,
                     const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                     const int64_t *ge_j, const int64_t *ge_w, const double *lam,
                     const double *delta, const int64_t *period, int64_t profile_stride,
                     double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                     int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                     int rng_mode, uint64_t rng_seed, int64_t first_trial, const double *native_sig,
                     pbsa_plan **out) {
    return guarded([&] {
        if (!out) fail(PBSA_EINVAL, "null plan out-pointer");
        *out = nullptr;
        if (mm < 0 || gm < 0) fail(PBSA_EINVAL, "negative edge count");
        std::unique_ptr<pbsa_plan> P(new pbsa_plan());
        create_plan(*P, device, n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm, ge_i,
                    ge_j, ge_w, lam, delta, period, profile_stride, i0_min, beta, cycles, t_res,
                    algo, alpha, p_stall, trials, keys, rng_mode, rng_seed, first_trial, native_sig);
        DeviceGuard dg(device);
        P->mm_ = mm;
        P->gm_ = gm;
        // a one-shot call's plan is launched directly: instantiating a graph of
        // ~10^4 launch nodes (a timing spread, several chains) costs more than
        // launching them once
        if (g_oneshot && !P->pipelined) P->direct = true;
        if (P->pipelined || P->direct) {  // one-shot: launched directly (or captured with its outputs) by the call
            *out = P.release();
            return;
        }
        // capture the whole anneal into one graph
        CK(cudaStreamBeginCapture(P->stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_run(*P, mm, gm);
        } catch (...) {
            cudaGraph_t g;
            cudaStreamEndCapture(P->stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t graph;
        CK(cudaStreamEndCapture(P->stream, &graph));
        cudaError_t e = cudaGraphInstantiate(&P->graph_exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(e);
        *out = P.release();
    });
}
}  // namespace

extern "C" {

int pbsa_plan_create_ex(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                        const double *values, const double *h, int64_t mm, const int64_t *me_i,
                        const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                        const int64_t *ge_j, const int64_t *ge_w, const double *lam,
                        const double *delta, const int64_t *period, int64_t profile_stride,
                        double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                        int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                        int rng_mode, uint64_t rng_seed, int64_t first_trial, pbsa_plan **out) {
    return plan_create_impl(device, n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm, ge_i, ge_j,
                            ge_w, lam, delta, period, profile_stride, i0_min, beta, cycles, t_res, algo,
                            alpha, p_stall, trials, keys, rng_mode, rng_seed, first_trial, nullptr, out);
}

int pbsa_plan_create_np(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                        const double *values, const double *h, int64_t mm, const int64_t *me_i,
                        const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                        const int64_t *ge_j, const int64_t *ge_w, const double *native_sigmas,
                        double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                        int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                        uint64_t rng_seed, int64_t first_trial, pbsa_plan **out) {
    if (!native_sigmas) {
        g_last_error = "null native_sigmas";
        return PBSA_EINVAL;
    }
    return plan_create_impl(device, n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm, ge_i, ge_j,
                            ge_w, nullptr, nullptr, nullptr, 0, i0_min, beta, cycles, t_res, algo, alpha,
                            p_stall, trials, keys, PBSA_RNG_PHILOX, rng_seed, first_trial, native_sigmas,
                            out);
}

int pbsa_plan_run(pbsa_plan *P, float *device_ms) {
    return guarded([&] {
        if (!P) fail(PBSA_EINVAL, "null plan");
        DeviceGuard dg(P->device);
        CK(cudaEventRecord(P->ev_start, P->stream));
        launch_run(*P);
        CK(cudaEventRecord(P->ev_end, P->stream));
        CK(cudaEventSynchronize(P->ev_end));
        P->ran = true;
        if (device_ms) CK(cudaEventElapsedTime(device_ms, P->ev_start, P->ev_end));
    });
}

int pbsa_plan_info(const pbsa_plan *P, int *path, int64_t *launches_per_run,
                   double *sweep_ms_mean, int64_t *sweep_launches, int64_t *words) {
    return guarded([&] {
        if (!P) fail(PBSA_EINVAL, "null plan");
        if (path) *path = P->path;
        if (launches_per_run) *launches_per_run = P->launches;
        if (sweep_launches) *sweep_launches = P->sweep_launches;
        if (words) *words = P->W;
        if (sweep_ms_mean) {
            *sweep_ms_mean = 0.0;
            if (P->ran && P->sweep_launches) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, P->ev_sweep0, P->ev_sweep1));
                // the packed phase also holds the final cut-only pass
                const int64_t k = P->path == PBSA_PATH_PACKED ? P->sweep_launches + 1
                                                               : P->sweep_launches;
                *sweep_ms_mean = (double)ms / (double)k;
            }
        }
    });
}

int pbsa_plan_kernel(const pbsa_plan *P, int *kernel, int *cluster_size) {
    return guarded([&] {
        if (!P) fail(PBSA_EINVAL, "null plan");
        int k;
        if (P->path == PBSA_PATH_PACKED)
            k = P->resident ? (P->res_timing ? PBSA_KERNEL_RESIDENT_TIMING : PBSA_KERNEL_RESIDENT)
                            : (P->var_mode && !P->var_uniform ? (P->bucket ? PBSA_KERNEL_PACKED_BUCKET : PBSA_KERNEL_PACKED_TIMING)
                                                                : PBSA_KERNEL_PACKED);
        else
            k = P->active_mode ? (P->fast ? PBSA_KERNEL_ACTIVE_FAST : PBSA_KERNEL_ACTIVE) : PBSA_KERNEL_FULL;
        if (kernel) *kernel = k;
        if (cluster_size) *cluster_size = P->resident ? P->res_cs : 1;
    });
}

int pbsa_plan_summary(pbsa_plan *P, int64_t *final_cut_sum, int64_t *best_cut_max,
                      int64_t *updates) {
    return guarded([&] {
        if (!P) fail(PBSA_EINVAL, "null plan");
        if (!P->ran) fail(PBSA_EINVAL, "plan has not been run");
        DeviceGuard dg(P->device);
        std::vector<int64_t> last(P->T), best(P->T);
        // last-cycle cut of every trial: column C-1 of [T][C]
        CK(cudaMemcpy2DAsync(last.data(), sizeof(int64_t), P->trace_cut.p + (P->cycles - 1),
                             P->cycles * sizeof(int64_t), sizeof(int64_t), P->T,
                             cudaMemcpyDeviceToHost, P->stream));
        CK(cudaMemcpyAsync(best.data(), P->best.p, P->T * sizeof(int64_t), cudaMemcpyDeviceToHost,
                           P->stream));
        CK(cudaStreamSynchronize(P->stream));
        int64_t s = 0, b = -(1LL << 62);
        for (int64_t t = 0; t < P->T; ++t) {
            s += last[t];
            b = std::max(b, best[t]);
        }
        if (final_cut_sum) *final_cut_sum = s;
        if (best_cut_max) *best_cut_max = b;
        if (updates) *updates = P->updates_per_run;
    });
}

int pbsa_plan_download(pbsa_plan *P, int8_t *spins, double *inputs, double *hist, int64_t *counts,
                       double *trace_i0, double *trace_energy, int64_t *trace_cut,
                       int64_t *best_cut) {
    return guarded([&] {
        download_impl(P, spins, inputs, hist, counts, trace_i0, trace_energy, trace_cut, best_cut,
                      false);
    });
}

}  // extern "C"

namespace pbsa_rt {

// Outputs that do not depend on the run: the i0 trace, zero histories of the
// rules that keep none, and update counts fixed by the periods.  The one-shot
// call writes them on the host while the device anneals.
void host_constant_outputs(pbsa_plan *P, double *hist, int64_t *counts, double *trace_i0) {
    const int64_t n = P->n, T = P->T, C = P->cycles;
    if (trace_i0)
        for (int64_t t = 0; t < T; ++t) std::memcpy(trace_i0 + t * C, P->i0.data(), C * sizeof(double));
    if (P->path == PBSA_PATH_PACKED) {
        if (hist && !P->tapsa_hist_from_raw && !P->tapsa_packed)
            parallel_fill(hist, (size_t)(T * n * P->alpha), 0.0);
        if (counts && P->pcl.empty()) {
            parallel_fill(counts, (size_t)(T * n), (int64_t)C);  // every p-bit fires once per cycle
        } else if (counts) {  // timing spread: #{count < C t_res : period | count}
            const int64_t mc = C * P->t_res;
            const uint8_t *pc = P->pcl.data();
            parallel_for(T * n, 1 << 20, [&](int64_t lo, int64_t hi) {
                for (int64_t k = lo; k < hi; ++k) counts[k] = (mc + pc[k] - 1) / pc[k];
            });
        }
    } else {
        if (hist && P->algo != 1) parallel_fill(hist, (size_t)(T * n * P->alpha), 0.0);
        if (counts && P->fast) {  // fast active mode: #{count < C t_res : period | count}
            const int64_t mc = C * P->t_res;
            const int32_t *pc = P->apcl.data();
            parallel_for(T * n, 1 << 20, [&](int64_t lo, int64_t hi) {
                for (int64_t k = lo; k < hi; ++k) counts[k] = (mc + pc[k] - 1) / pc[k];
            });
        }
    }
}

void download_impl(pbsa_plan *P, int8_t *spins, double *inputs, double *hist, int64_t *counts,
                   double *trace_i0, double *trace_energy, int64_t *trace_cut, int64_t *best_cut,
                   bool consts_done) {
    {
        if (!P) fail(PBSA_EINVAL, "null plan");
        if (!P->ran) fail(PBSA_EINVAL, "plan has not been run");
        DeviceGuard dg(P->device);
        cudaStream_t st = P->stream;
        const int64_t n = P->n, T = P->T, C = P->cycles;
        const int TB = 256;
        if (trace_cut)
            CK(cudaMemcpyAsync(trace_cut, P->trace_cut.p, T * C * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
        if (trace_energy)
            CK(cudaMemcpyAsync(trace_energy, P->trace_energy.p, T * C * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
        if (best_cut)
            CK(cudaMemcpyAsync(best_cut, P->best.p, T * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        AllocStream as(st);
        DevBuf<int8_t> dspins;
        DevBuf<double> dinputs, dhist;
        DevBuf<int32_t> dcounts;
        DevBuf<int64_t> dcounts64;
        if (P->path == PBSA_PATH_PACKED) {
            if (spins) {
                dspins.alloc((size_t)T * n);
                pbsa::unpack_spins<<<grid_for(n * T, TB), TB, 0, st>>>(
                    P->p_spins[P->final_parity].p, dspins.p, (int)n, (int)P->W, (int)T);
            }
            const double f_last = P->tapsa_packed ? (double)std::min<int64_t>(C, P->alpha) : 1.0;
            if (inputs && !P->var_mode) {
                dinputs.alloc((size_t)T * n);
                if (P->spsa_packed)
                    pbsa::inputs_from_sidx<<<grid_for(n * T, TB), TB, 0, st>>>(
                        P->sidx.p, P->i0_dev.p, dinputs.p, (int)n, (int)T, P->K, P->dmax);
                else
                    pbsa::inputs_from_raw<<<grid_for(n * T, TB), TB, 0, st>>>(
                        P->raw_last.p, dinputs.p, P->i0[C - 1], (int)n, (int)P->Tp, (int)T, f_last);
            }
            if (hist && P->tapsa_hist_from_raw) {
                // TAPSA with alpha = 1: the history holds the last raw field
                dhist.alloc((size_t)T * n);
                pbsa::inputs_from_raw<<<grid_for(n * T, TB), TB, 0, st>>>(
                    P->raw_last.p, dhist.p, 1.0, (int)n, (int)P->Tp, (int)T, 1.0);
            }
            if (hist && P->tapsa_packed) {
                dhist.alloc((size_t)T * n * P->alpha);
                const int written = (int)std::min<int64_t>(C, P->alpha);
                switch (P->L) {
                    case 1: launch_hist_from_ring<1>(P->ring.p, P->rowptr.p, (int)n, (int)T, (int)P->alpha, written, dhist.p, st); break;
                    case 2: launch_hist_from_ring<2>(P->ring.p, P->rowptr.p, (int)n, (int)T, (int)P->alpha, written, dhist.p, st); break;
                    case 3: launch_hist_from_ring<3>(P->ring.p, P->rowptr.p, (int)n, (int)T, (int)P->alpha, written, dhist.p, st); break;
                    case 4: launch_hist_from_ring<4>(P->ring.p, P->rowptr.p, (int)n, (int)T, (int)P->alpha, written, dhist.p, st); break;
                    case 5: launch_hist_from_ring<5>(P->ring.p, P->rowptr.p, (int)n, (int)T, (int)P->alpha, written, dhist.p, st); break;
                    case 6: launch_hist_from_ring<6>(P->ring.p, P->rowptr.p, (int)n, (int)T, (int)P->alpha, written, dhist.p, st); break;
                    default: launch_hist_from_ring<7>(P->ring.p, P->rowptr.p, (int)n, (int)T, (int)P->alpha, written, dhist.p, st); break;
                }
            }
            // copies first (asynchronous into page-locked buffers), then the
            // host-side constant outputs while the DMA and kernels run
            if (spins) CK(cudaMemcpyAsync(spins, dspins.p, T * n, cudaMemcpyDeviceToHost, st));
            if (inputs)  // VAR: i0 * raw of each p-bit's last update, already [T][n]
                CK(cudaMemcpyAsync(inputs, P->var_mode ? P->inp_var.p : dinputs.p, T * n * sizeof(double),
                                   cudaMemcpyDeviceToHost, st));
            if (hist && (P->tapsa_hist_from_raw || P->tapsa_packed))
                CK(cudaMemcpyAsync(hist, dhist.p, T * n * (P->tapsa_packed ? P->alpha : 1) * sizeof(double),
                                   cudaMemcpyDeviceToHost, st));
            if (!consts_done) host_constant_outputs(P, hist, counts, trace_i0);
            CK(cudaStreamSynchronize(st));
        } else {
            dim3 tb(32, 8);
            if (spins) {
                dspins.alloc((size_t)T * n);
                dim3 g((unsigned)grid_for(T, 32), (unsigned)grid_for(n, 32));
                pbsa::transpose_tile<int8_t><<<g, tb, 0, st>>>(P->g_spins[P->final_parity].p,
                                                               dspins.p, (int)n, (int)P->Tp, (int)T);
            }
            const int64_t Np = (int64_t)P->alist.n;
            const int tsh = P->tshift;
            if (inputs) {
                dinputs.alloc((size_t)T * n);
                if (P->active_mode) {
                    pbsa::list_to_trial_major<double, double><<<grid_for(Np, TB), TB, 0, st>>>(
                        P->a_inputs.p, P->alist.p, Np, tsh, P->tmask, (int)n, 1, dinputs.p);
                } else {
                    dim3 g((unsigned)grid_for(T, 32), (unsigned)grid_for(n, 32));
                    pbsa::transpose_tile<double><<<g, tb, 0, st>>>(P->inputs.p, dinputs.p, (int)n,
                                                                   (int)P->Tp, (int)T);
                }
            }
            if (counts && !P->fast) {
                dcounts64.alloc((size_t)T * n);
                if (P->active_mode) {
                    pbsa::list_to_trial_major<int32_t, int64_t><<<grid_for(Np, TB), TB, 0, st>>>(
                        P->a_counts.p, P->alist.p, Np, tsh, P->tmask, (int)n, 1, dcounts64.p);
                } else {
                    dcounts.alloc((size_t)T * n);
                    dim3 g((unsigned)grid_for(T, 32), (unsigned)grid_for(n, 32));
                    pbsa::transpose_tile<int32_t><<<g, tb, 0, st>>>(P->counts.p, dcounts.p, (int)n,
                                                                    (int)P->Tp, (int)T);
                    pbsa::widen_i32<<<grid_for(T * n, TB), TB, 0, st>>>(dcounts.p, dcounts64.p, T * n);
                }
            }
            if (hist && P->algo == 1) {
                const int64_t rows = n * P->alpha;
                dhist.alloc((size_t)T * rows);
                dim3 g((unsigned)grid_for(T, 32), (unsigned)grid_for(rows, 32));
                if (P->active_mode) {  // integer ring -> fp64 (exact: the raws are integers)
                    pbsa::list_to_trial_major<int32_t, double><<<grid_for(Np, TB), TB, 0, st>>>(
                        P->hist_i.p, P->alist.p, Np, tsh, P->tmask, (int)n, (int)P->alpha, dhist.p);
                } else {
                    pbsa::transpose_tile<double><<<g, tb, 0, st>>>(P->hist.p, dhist.p, (int)rows,
                                                                   (int)P->Tp, (int)T);
                }
            }
            if (spins) CK(cudaMemcpyAsync(spins, dspins.p, T * n, cudaMemcpyDeviceToHost, st));
            if (inputs)
                CK(cudaMemcpyAsync(inputs, dinputs.p, T * n * sizeof(double), cudaMemcpyDeviceToHost, st));
            if (counts && !P->fast)
                CK(cudaMemcpyAsync(counts, dcounts64.p, T * n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            if (hist && P->algo == 1)
                CK(cudaMemcpyAsync(hist, dhist.p, T * n * P->alpha * sizeof(double),
                                   cudaMemcpyDeviceToHost, st));
            if (!consts_done) host_constant_outputs(P, hist, counts, trace_i0);
            CK(cudaStreamSynchronize(st));
        }
        CK(cudaGetLastError());
    }
}

}  // namespace

extern "C" {

int pbsa_plan_layout(const pbsa_plan *P, int64_t *phase_words, int *chains, int *warps_per_word,
                     int *hash_cache) {
    return guarded([&] {
        if (!P) fail(PBSA_EINVAL, "null plan");
        if (phase_words) *phase_words = P->phase_words;
        if (chains) *chains = (int)P->chain_streams.size() + 1;
        if (warps_per_word) *warps_per_word = P->warps_per_word;
        if (hash_cache) *hash_cache = P->use_cache ? 1 : 0;
    });
}

int pbsa_plan_bytes(const pbsa_plan *P, int64_t *h2d_bytes, int64_t *d2h_bytes) {
    return guarded([&] {
        if (!P) fail(PBSA_EINVAL, "null plan");
        const size_t up = P->p_spins[0].bytes_up + P->rowptr.bytes_up + P->adj.bytes_up + P->adj16.bytes_up + P->kfc.bytes_up +
                          P->thr.bytes_up + P->krg.bytes_up + P->col.bytes_up + P->me_i.bytes_up +
                          P->me_j.bytes_up + P->ge_i.bytes_up + P->ge_j.bytes_up +
                          P->val.bytes_up + P->h.bytes_up + P->me_w.bytes_up + P->lam.bytes_up +
                          P->delta.bytes_up + P->me_wi.bytes_up + P->h_int.bytes_up +
                          P->ge_w.bytes_up + P->period.bytes_up + P->kr.bytes_up +
                          P->kst.bytes_up + P->kspin.bytes_up + P->prof.bytes_up + P->lam64.bytes_up +
                          P->del64.bytes_up + P->pplanes.bytes_up + P->vdivs.bytes_up +
                          P->kfs.bytes_up + P->kstg.bytes_up + P->vali.bytes_up + P->hi32.bytes_up +
                          P->alist.bytes_up + P->adesc.bytes_up + P->athr.bytes_up + P->i0_dev.bytes_up +
                          P->ge_w32.bytes_up + P->me_w32.bytes_up + P->prof16.bytes_up;
        const int64_t T = P->T, n = P->n, C = P->cycles;
        int64_t down = T * n + T * n * 8 + 2 * T * C * 8 + T * 8;  // spins, inputs, traces, best
        if (P->path == PBSA_PATH_GENERAL) {
            down += T * n * 8;                                        // counts (int64)
            if (P->algo == 1) down += T * n * P->alpha * 8;           // history
        } else if (P->tapsa_hist_from_raw) {
            down += T * n * 8;
        } else if (P->tapsa_packed) {
            down += T * n * P->alpha * 8;
        }
        if (h2d_bytes) *h2d_bytes = (int64_t)up;
        if (d2h_bytes) *d2h_bytes = down;
    });
}

int pbsa_plan_destroy(pbsa_plan *P) {
    return guarded([&] {
        if (!P) return;
        DeviceGuard dg(P->device);
        delete P;
    });
}

int pbsa_anneal_loop_batch(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                           const double *values, const double *h, int64_t mm,
                           const int64_t *me_i, const int64_t *me_j, const double *me_w,
                           int64_t gm, const int64_t *ge_i, const int64_t *ge_j,
                           const int64_t *ge_w, const double *lam, const double *delta,
                           const int64_t *period, int64_t profile_stride, double i0_min,
                           double beta, int64_t cycles, int64_t t_res, int algo, int64_t alpha,
                           double p_stall, int64_t trials, const uint64_t *keys, int8_t *spins,
                           double *inputs, double *hist, int64_t *counts, double *trace_i0,
                           double *trace_energy, int64_t *trace_cut, int64_t *best_cut,
                           float *device_ms) {
    return pbsa_anneal_loop_batch_ex(device, n, indptr, indices, values, h, mm, me_i, me_j, me_w,
                                     gm, ge_i, ge_j, ge_w, lam, delta, period, profile_stride,
                                     i0_min, beta, cycles, t_res, algo, alpha, p_stall, trials,
                                     keys, PBSA_RNG_REPLAY, 0, 0, spins, inputs, hist, counts,
                                     trace_i0, trace_energy, trace_cut, best_cut, device_ms);
}

}  // extern "C"

