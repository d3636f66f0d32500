/*
 * pbsa.h -- C ABI of the B200-native p-bit simulated-annealing sweep.
 *
 * Drop-in boundary for the reference's one hot loop,
 *   pbitsa._kernels.anneal_loop(indptr, indices, values, h, me_i, me_j, me_w,
 *                               ge_i, ge_j, ge_w, lam, delta, period, i0_min,
 *                               beta, cycles, t_res, algo, alpha, p_stall, key)
 *   (/root/reference/pkg/src/pbitsa/_kernels.py:68-175, called from
 *    annealer.run_anneal, annealer.py:216-238, one trial per call)
 * generalised to T independent trials per call, which is how
 * engine.run_trials (engine.py:82-127) fans it out.  Every argument keeps the
 * reference's meaning and dtype; outputs are the same 8 arrays stacked over
 * trials.  Plain pointers and sizes only; all buffers are HOST memory unless
 * a function says otherwise.  Every function returns PBSA_OK (0) or a
 * negative status; pbsa_last_error() then describes the failure (thread-local).
 * Thread-safe: no global mutable state; a plan is used by one thread at a time.
 */
#ifndef PBSA_H
#define PBSA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBSA_ABI_VERSION 1

enum {
    PBSA_OK = 0,
    PBSA_EINVAL = -1, /* invalid argument (ValueError on the Python side) */
    PBSA_ECUDA = -2,  /* CUDA runtime error                                */
    PBSA_ENOMEM = -3, /* host or device allocation failed                  */
};

/* Input rule codes, identical to _kernels.py:38-41 (ALGO_PSA/TAPSA/SPSA). */
enum { PBSA_ALGO_PSA = 0, PBSA_ALGO_TAPSA = 1, PBSA_ALGO_SPSA = 2 };

/* Which device path a plan runs (pbsa_plan_info). */
enum { PBSA_PATH_PACKED = 1, PBSA_PATH_GENERAL = 2 };

/* Random stream of the activation draws (pbsa_plan_create_ex). */
enum {
    PBSA_RNG_REPLAY = 0, /* the reference's counter hash (streams.py:29-55), bit-exact */
    PBSA_RNG_PHILOX = 1  /* native Philox4x32-10 (philox.cuh): X = philox({i, count,
                            k >> 2, 3}, rng_seed)[k & 3] for global trial k, and
                            r = (2X + 1) 2^-32 - 1 */
};

typedef struct pbsa_plan pbsa_plan;

int pbsa_abi_version(void);
const char *pbsa_last_error(void);
int pbsa_device_count(int *count);

/*
 * Upload one batch of trials to `device` and build its device-resident
 * state (CSR adjacency, per-trial key prefixes, profiles, schedule tables).
 *
 *   n, indptr[n+1], indices[nnz], values[nnz], h[n]      IsingModel CSR
 *        (model.py:21-33, 84-128; int64 / float64 exactly as the reference)
 *   mm, me_i/me_j[mm], me_w[mm]                          model edges (energy)
 *   gm, ge_i/ge_j/ge_w[gm]                               graph edges (cut);
 *        gm = 0 means "no graph" (annealer.py:208-213): cut outputs are 0
 *   lam, delta (float64), period (int64)                 VariabilityProfile;
 *        rows of n, `profile_stride` = 0 (one profile shared by all trials)
 *        or n (row t belongs to trial t).  NULL for all three = ideal.
 *   i0_min, beta, cycles, t_res                          AnnealSchedule
 *   algo, alpha, p_stall                                 AlgorithmConfig
 *        (alpha = 1 unless TAPSA, annealer.py:235)
 *   trials, keys[trials]                                 run_key(seed) per trial
 *        (streams.py:58-60)
 */
int pbsa_plan_create(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                     const double *values, const double *h, int64_t mm, const int64_t *me_i,
                     const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                     const int64_t *ge_j, const int64_t *ge_w, const double *lam,
                     const double *delta, const int64_t *period, int64_t profile_stride,
                     double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                     int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                     pbsa_plan **out);

/*
 * pbsa_plan_create with a choice of random stream.  rng_mode PBSA_RNG_REPLAY
 * is pbsa_plan_create.  PBSA_RNG_PHILOX draws every activation uniform from
 * Philox4x32-10 keyed by rng_seed, with the global trial index
 * first_trial + t in the counter (a multiple of 4, so any sharding of the
 * trials by multiples of 4 gives identical per-trial results); initial spins
 * still come from keys[] as in the reference; the SpSA stall draw is the same
 * Philox word with tag 4.  Philox mode covers every input of the packed path
 * (+-1 MAX-CUT models of degree <= 127: all three rules on an ideal profile,
 * the plain rule with a lam/delta/period profile); other inputs return
 * PBSA_EINVAL.  No reference interface corresponds: the
 * reference has only its counter hash (streams.py); this is the north_star's
 * native RNG mode.
 */
int pbsa_plan_create_ex(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                        const double *values, const double *h, int64_t mm, const int64_t *me_i,
                        const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                        const int64_t *ge_j, const int64_t *ge_w, const double *lam,
                        const double *delta, const int64_t *period, int64_t profile_stride,
                        double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                        int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                        int rng_mode, uint64_t rng_seed, int64_t first_trial, pbsa_plan **out);

/*
 * Run the whole anneal on the device from the initial spins: `cycles` main
 * cycles of `t_res` synchronous sub-steps each, per-cycle energy/cut traces.
 * Inputs are already resident; nothing crosses PCIe.  *device_ms (optional)
 * receives the CUDA-event time of the run on the plan's stream.
 */
int pbsa_plan_run(pbsa_plan *plan, float *device_ms);

/*
 * Copy the results of the last run back, in anneal_loop's return order
 * (_kernels.py:175), stacked over trials (row t = trial t):
 *   spins[T*n] int8, inputs[T*n] f64, hist[T*n*alpha] f64, counts[T*n] i64,
 *   trace_i0[T*cycles] f64, trace_energy[T*cycles] f64,
 *   trace_cut[T*cycles] i64, best_cut[T] i64.
 * Any output pointer may be NULL to skip it.
 */
int pbsa_plan_download(pbsa_plan *plan, int8_t *spins, double *inputs, double *hist,
                       int64_t *counts, double *trace_i0, double *trace_energy,
                       int64_t *trace_cut, int64_t *best_cut);

/*
 * Device-side summary of the last run without downloading traces:
 * final_cut_sum = sum over trials of the last-cycle cut, best_cut_max = max
 * over trials of best cut, updates = total p-bit updates performed.
 */
int pbsa_plan_summary(pbsa_plan *plan, int64_t *final_cut_sum, int64_t *best_cut_max,
                      int64_t *updates);

/*
 * Plan facts: path (PBSA_PATH_*), launches per run, the dominant sweep
 * kernel's mean per-launch time of the last run in ms (CUDA events on the
 * plan stream) and its launch count, and the trial-word count.
 */
int pbsa_plan_info(const pbsa_plan *plan, int *path, int64_t *launches_per_run,
                   double *sweep_ms_mean, int64_t *sweep_launches, int64_t *words);

/* Which sweep kernel a plan runs (pbsa_plan_kernel). */
enum {
    PBSA_KERNEL_PACKED = 1,          /* packed_sweep, one launch per sub-step */
    PBSA_KERNEL_PACKED_TIMING = 2,   /* packed_sweep_timing (period spread) */
    PBSA_KERNEL_RESIDENT = 3,        /* resident_sweep, one cluster launch per run */
    PBSA_KERNEL_RESIDENT_TIMING = 4, /* resident_timing */
    PBSA_KERNEL_ACTIVE_FAST = 5,     /* general path: active lists, plain rule */
    PBSA_KERNEL_ACTIVE = 6,          /* general path: active lists, all rules */
    PBSA_KERNEL_FULL = 7,            /* general path: fp64 full pass */
    PBSA_KERNEL_PACKED_BUCKET = 8    /* packed_sweep_bucket (period spread, period-sorted slots) */
};

/*
 * The sweep kernel family of a plan (PBSA_KERNEL_*), and the cluster size of
 * the resident kernels (1 otherwise).  Diagnostic; results do not depend on it.
 */
int pbsa_plan_kernel(const pbsa_plan *plan, int *kernel, int *cluster_size);

/*
 * Launch shape of a launched (non-resident) packed plan: word-phase width in
 * words (phases run one after another; = words when unphased), concurrent
 * word-group chains per phase, warps per trial word, and whether the
 * per-(trial, node) first-absorb hash cache is used.  Diagnostic: the parity
 * tests assert that they exercise the shape the benchmark times.
 */
int pbsa_plan_layout(const pbsa_plan *plan, int64_t *phase_words, int *chains,
                     int *warps_per_word, int *hash_cache);

/*
 * Bytes one end-to-end call moves: host->device at plan creation (CSR,
 * edges, keys, profiles, schedule tables) and device->host for a full
 * pbsa_plan_download of all eight outputs.
 */
int pbsa_plan_bytes(const pbsa_plan *plan, int64_t *h2d_bytes, int64_t *d2h_bytes);

int pbsa_plan_destroy(pbsa_plan *plan);

/*
 * One-shot batched anneal_loop: create + run + download + destroy, all host
 * buffers (the end-to-end path engine.run_trials / annealer.run_anneal use).
 * Output layout as pbsa_plan_download; *device_ms as pbsa_plan_run.
 */
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
                           float *device_ms);

/*
 * Native variability profiles (Philox stream only; no reference counterpart):
 * instead of lam/delta/period arrays the caller gives the three standard
 * deviations native_sigmas = {sigma_lambda, sigma_delta, sigma_nu} of
 * pbit.py:57-75 and the plan draws every p-bit's profile on the device from
 * Philox4x32-10 (counter (node, trial_hi, trial_lo, 5) under rng_seed, two
 * Box-Muller pairs): lam = 1 + s_l z1, delta = s_d z2, period = max(1,
 * rint(t_res (1 + s_n z3))).  No host sampling, no profile upload; the
 * packed path's plain rule only (else -1).  pbsa_native_profiles returns the
 * profiles a plan with the same seed and first_trial draws (periods clamped
 * to cycles * t_res, which fires identically).
 */
int pbsa_plan_create_np(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                        const double *values, const double *h, int64_t mm, const int64_t *me_i,
                        const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                        const int64_t *ge_j, const int64_t *ge_w, const double *native_sigmas,
                        double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                        int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                        uint64_t rng_seed, int64_t first_trial, pbsa_plan **out);
int pbsa_anneal_loop_batch_np(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                              const double *values, const double *h, int64_t mm, const int64_t *me_i,
                              const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                              const int64_t *ge_j, const int64_t *ge_w, const double *native_sigmas,
                              double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                              int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                              uint64_t rng_seed, int64_t first_trial, int8_t *spins, double *inputs,
                              double *hist, int64_t *counts, double *trace_i0, double *trace_energy,
                              int64_t *trace_cut, int64_t *best_cut, float *device_ms);
int pbsa_native_profiles(int device, uint64_t rng_seed, int64_t first_trial, int64_t trials, int64_t n,
                         int64_t t_res, int64_t cycles, const double *native_sigmas, double *lam,
                         double *delta, int64_t *period);

/*
 * One-shot calls of the plain rule whose output buffers are page-locked keep
 * their plan (device buffers, the captured graph with per-phase output copies)
 * for the next call of the same shape; each call still uploads every input
 * and writes every output.  PBSA_PLAN_CACHE=0 disables this; this frees the
 * cached plans.
 */
int pbsa_plan_cache_clear(void);

/* Host<->device bytes of the calling thread's last one-shot call. */
int pbsa_last_call_bytes(int64_t *h2d_bytes, int64_t *d2h_bytes);

/* pbsa_anneal_loop_batch with a choice of random stream (see pbsa_plan_create_ex). */
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
                              float *device_ms);

/*
 * pbsa_anneal_loop_batch_ex over a device-ordinal list (the
 * reference's engine.run_trials fan-out, engine.py:119-123): the trials are
 * split into ndev contiguous shards (interior edges multiples of 4, so the
 * Philox stream's four-trial groups never straddle a shard), shard r runs on
 * devices[r] from its own host thread with its own plan and stream, and every
 * output lands at its trial's row of the caller's buffers -- identical to the
 * single-device call.  A device may be listed more than once.  *device_ms is
 * the largest shard's device time; the first failing shard's code is returned.
 */
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
                                   int64_t *best_cut, float *device_ms);

/*
 * Device self-checks (used by the parity tests): evaluate the device
 * counter hash stream_u64(key, tag, a, b) (streams.py:41-45) and the device
 * tanh on `count` host inputs.
 */
int pbsa_debug_stream_u64(int device, int64_t count, const uint64_t *key, const uint64_t *tag,
                          const uint64_t *a, const uint64_t *b, uint64_t *out);
int pbsa_debug_tanh(int device, int64_t count, const double *x, double *out);
/* The varied-profile prefilter on given (lam, delta, i0, raw, zh): out bit 1 =
 * undecided (exact fp64 recheck), bit 0 = the decision otherwise. */
int pbsa_debug_var_prefilter(int device, int64_t count, const double *lam, const double *delta,
                             const double *i0, const int *raw, const uint32_t *zh, uint32_t *out);
/* Philox4x32-10 on the device: ctr[4*count], key[2*count] -> out[4*count]. */
int pbsa_debug_philox(int device, int64_t count, const uint32_t *ctr, const uint32_t *key,
                      uint32_t *out);

/*
 * Text of the reference CLI's trace CSV rows (cli.py:163-168, no header) for
 * T trials x C cycles: "t,c,<i0 text c>,<energy>.0,<cut>\n" with the caller's
 * repr() strings of the (shared) i0 trace in i0_text[i0_off[c] .. i0_off[c+1]),
 * integral energies energy[T*C] (|E| < 1e16, so repr is the digits + ".0")
 * and cut[T*C] (NULL: empty column).  *out_len receives the byte count;
 * PBSA_EINVAL if out_cap is too small.  Host threads, no GPU.
 */
int pbsa_format_trace_csv(int64_t T, int64_t C, const char *i0_text, const int64_t *i0_off,
                          const int64_t *energy, const int64_t *cut, char *out, int64_t out_cap,
                          int64_t *out_len);

/* Host builds of device-side pieces (no GPU needed):
 *   pbsa_libm_tanh_host  -- the device tanh (same source, libm_tanh.cuh);
 *   pbsa_threshold_host  -- the packed path's activation threshold for a
 *     tanh value t: the update is +1 iff hash >= threshold, exactly when
 *     r + t >= 0 with r = 2 u01 - 1 (_kernels.py:149-152); ~0 means never. */
double pbsa_libm_tanh_host(double x);
uint64_t pbsa_threshold_host(double t);
/*   pbsa_threshold_native_host -- the same for the Philox stream: +1 iff the
 *     32-bit draw X >= threshold (2^32 means never);
 *   pbsa_philox_host -- Philox4x32-10 of ctr[4] under key[2] (same source as
 *     the device, philox.cuh). */
uint64_t pbsa_threshold_native_host(double t);
void pbsa_philox_host(const uint32_t *ctr, const uint32_t *key, uint32_t *out);
/*   pbsa_choose_phases_host -- the packed sweep's word-phase width for a batch
 *     of W words of `chunks` 32-node chunks on a device with resident_warps
 *     resident sweep warps and an L2 budget in bytes (0: one phase), as plan
 *     creation picks it (csrc/plan.cu choose_phases); *balance receives
 *     whether the chunks are spread evenly over fewer warps. */
int64_t pbsa_choose_phases_host(int64_t chunks, int64_t W, int64_t resident_warps, int64_t l2_budget,
                                int *balance);

#ifdef __cplusplus
}
#endif
#endif /* PBSA_H */
