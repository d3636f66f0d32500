/*
 * psa_oracle.c -- CPU restatement of the reference p-bit annealing loop.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path links, loads or
 * calls this file: it is the checker used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * leg.  The product is the CUDA library in paper_2601_14476_b200/csrc/.
 *
 * Parity pinned: the outputs of this restatement are checked bit-for-bit
 * against golden vectors produced by the reference package itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/pbitsa and
 * records its outputs; tests/test_oracle_golden.py replays them here).
 *
 * What it restates (all citations relative to /root/reference/pkg/src/pbitsa):
 *   - counter hash            streams.py:29-55, _kernels.py:44-59
 *   - anneal_loop              _kernels.py:68-175 (all three input rules)
 *   - per-cycle energy / cut   _kernels.py:157-171 (same accumulation order)
 *   - and, with no reference counterpart, the native Philox4x32-10 activation
 *     stream of the CUDA library's PBSA_RNG_PHILOX mode (pinned by the
 *     published Random123 known-answer vectors, not by the reference)
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (see oracle/Makefile).
 * FMA contraction must stay off so that every fp64 operation rounds exactly
 * as the numba-compiled reference (fastmath off, _kernels.py:15-16) does.
 * tanh comes from the system libm, exactly like the reference (_kernels.py:150).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_GAMMA 0x9E3779B97F4A7C15ULL
#define ORC_M1 0xBF58476D1CE4E5B9ULL
#define ORC_M2 0x94D4A04C32684F87ULL

enum { ORC_TAG_RUN = 1, ORC_TAG_SPIN = 2, ORC_TAG_R = 3, ORC_TAG_STALL = 4,
       ORC_TAG_TRIAL = 5, ORC_TAG_PROFILE = 6 };
enum { ORC_PSA = 0, ORC_TAPSA = 1, ORC_SPSA = 2 };

/* splitmix64 finaliser -- streams.py:29-34 */
uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * ORC_M1;
    z = (z ^ (z >> 27)) * ORC_M2;
    return z ^ (z >> 31);
}

/* streams.py:37-38 */
uint64_t orc_absorb(uint64_t h, uint64_t w) { return orc_mix64((h + ORC_GAMMA) ^ w); }

/* streams.py:41-45 */
uint64_t orc_stream_u64(uint64_t key, uint64_t tag, uint64_t a, uint64_t b) {
    return orc_absorb(orc_absorb(orc_absorb(key, tag), a), b);
}

/* streams.py:48-50 / _kernels.py:56-59: top 53 bits scaled to [0, 1) */
double orc_u01(uint64_t key, uint64_t tag, uint64_t a, uint64_t b) {
    return (double)(orc_stream_u64(key, tag, a, b) >> 11) * 0x1p-53;
}

double orc_tanh(double x) { return tanh(x); }

/*
 * Native RNG mode (no reference counterpart: the north_star's Philox stream,
 * include/pbsa.h PBSA_RNG_PHILOX).  Philox4x32-10 as published by Salmon et
 * al. (SC'11, Random123): per round (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 * c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0), then k += (W0, W1).  Pinned by the
 * Random123 known-answer vectors in tests/test_oracle_golden.py.
 */
void orc_philox4x32_10(const uint32_t *ctr, const uint32_t *key, uint32_t *out) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The native stream's word X of global trial k: word (k & 3) of
 * Philox(ctr = {i, count, k >> 2, tag}, key = seed); tag 3 = activation,
 * 4 = SpSA stall. */
static uint32_t orc_native_x(uint64_t seed, uint64_t k, uint64_t i, uint64_t count, uint32_t tag) {
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)count, (uint32_t)(k >> 2), tag};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)}, o[4];
    orc_philox4x32_10(ctr, key, o);
    return o[k & 3];
}

/* Native activation: r = 2u - 1 with u = (X + 1/2) 2^-32, i.e. (2X + 1) 2^-32 - 1. */
static double orc_native_r(uint64_t seed, uint64_t k, uint64_t i, uint64_t count) {
    return (2.0 * (double)orc_native_x(seed, k, i, count, 3u) + 1.0) * 0x1p-32 - 1.0;
}

int orc_anneal_rng(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
                   const double *h, int64_t mm, const int64_t *me_i, const int64_t *me_j,
                   const double *me_w, int64_t gm, const int64_t *ge_i, const int64_t *ge_j,
                   const int64_t *ge_w, const double *lam, const double *delta,
                   const int64_t *period, double i0_min, double beta, int64_t cycles,
                   int64_t t_res, int algo, int64_t alpha, double p_stall, uint64_t key, int rng,
                   uint64_t seed, int64_t trial, int8_t *spins, double *inputs, double *hist,
                   int64_t *counts, double *trace_i0, double *trace_energy, int64_t *trace_cut,
                   int64_t *best_cut);

/*
 * One trial of the annealing loop (_kernels.py:68-175).
 *
 * Inputs mirror anneal_loop's positional arguments; outputs are caller-owned
 * buffers:  spins[n], inputs[n], hist[n*alpha], counts[n], trace_i0[cycles],
 * trace_energy[cycles], trace_cut[cycles], best_cut[1].
 * Returns 0, or -1 if scratch allocation failed.
 */
int orc_anneal(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
               const double *h, int64_t mm, const int64_t *me_i, const int64_t *me_j,
               const double *me_w, int64_t gm, const int64_t *ge_i, const int64_t *ge_j,
               const int64_t *ge_w, const double *lam, const double *delta,
               const int64_t *period, double i0_min, double beta, int64_t cycles, int64_t t_res,
               int algo, int64_t alpha, double p_stall, uint64_t key, int8_t *spins,
               double *inputs, double *hist, int64_t *counts, double *trace_i0,
               double *trace_energy, int64_t *trace_cut, int64_t *best_cut) {
    return orc_anneal_rng(n, indptr, indices, values, h, mm, me_i, me_j, me_w, gm, ge_i, ge_j,
                          ge_w, lam, delta, period, i0_min, beta, cycles, t_res, algo, alpha,
                          p_stall, key, 0, 0, 0, spins, inputs, hist, counts, trace_i0,
                          trace_energy, trace_cut, best_cut);
}

/* orc_anneal with a choice of activation stream: rng = 0 the reference's
 * counter hash, rng = 1 the native Philox draw of global trial `trial`
 * under `seed` (orc_native_r).  Everything else is identical. */
int orc_anneal_rng(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
                   const double *h, int64_t mm, const int64_t *me_i, const int64_t *me_j,
                   const double *me_w, int64_t gm, const int64_t *ge_i, const int64_t *ge_j,
                   const int64_t *ge_w, const double *lam, const double *delta,
                   const int64_t *period, double i0_min, double beta, int64_t cycles,
                   int64_t t_res, int algo, int64_t alpha, double p_stall, uint64_t key, int rng,
                   uint64_t seed, int64_t trial, int8_t *spins, double *inputs, double *hist,
                   int64_t *counts, double *trace_i0, double *trace_energy, int64_t *trace_cut,
                   int64_t *best_cut) {
    int64_t *stage_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int8_t *stage_val = (int8_t *)malloc((size_t)(n > 0 ? n : 1));
    if (!stage_idx || !stage_val) {
        free(stage_idx);
        free(stage_val);
        return -1;
    }
    /* initial spins: u01(key, TAG_SPIN, i, 0) < 0.5 -> +1   (_kernels.py:94-97) */
    for (int64_t i = 0; i < n; ++i)
        spins[i] = orc_u01(key, ORC_TAG_SPIN, (uint64_t)i, 0) < 0.5 ? 1 : -1;
    memset(inputs, 0, sizeof(double) * (size_t)n);
    memset(hist, 0, sizeof(double) * (size_t)(n * alpha));
    memset(counts, 0, sizeof(int64_t) * (size_t)n);
    int64_t best = -(((int64_t)1) << 62); /* _kernels.py:108 */

    /* _kernels.py:110-116: all periods == t_res -> only sub-step 0 can fire */
    int uniform = 1;
    for (int64_t i = 0; i < n; ++i)
        if (period[i] != t_res) { uniform = 0; break; }

    double i0 = i0_min;
    for (int64_t c = 0; c < cycles; ++c) {
        for (int64_t s = 0; s < t_res; ++s) {
            if (uniform && s != 0) continue;
            int64_t count = c * t_res + s;
            int64_t n_active = 0;
            for (int64_t i = 0; i < n; ++i) {
                if (count % period[i] != 0) continue;
                double raw = h[i];
                for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
                    raw += values[k] * (double)spins[indices[k]];
                double inp;
                if (algo == ORC_TAPSA) {
                    int64_t cnt = counts[i];
                    hist[i * alpha + cnt % alpha] = raw;
                    int64_t filled = cnt + 1 < alpha ? cnt + 1 : alpha;
                    double acc = 0.0;
                    for (int64_t q = 0; q < filled; ++q) acc += hist[i * alpha + q];
                    inp = i0 * (acc / (double)filled);
                } else if (algo == ORC_SPSA) {
                    if (counts[i] == 0) {
                        inp = i0 * raw;
                    } else {
                        double u = rng ? ((double)orc_native_x(seed, (uint64_t)trial, (uint64_t)i,
                                                                (uint64_t)count, 4u) + 0.5) * 0x1p-32
                                       : orc_u01(key, ORC_TAG_STALL, (uint64_t)i, (uint64_t)count);
                        inp = u < p_stall ? inputs[i] : i0 * raw;
                    }
                } else {
                    inp = i0 * raw;
                }
                inputs[i] = inp;
                counts[i] += 1;
                double r = rng ? orc_native_r(seed, (uint64_t)trial, (uint64_t)i, (uint64_t)count)
                               : 2.0 * orc_u01(key, ORC_TAG_R, (uint64_t)i, (uint64_t)count) - 1.0;
                double act = r + tanh(lam[i] * (inp + delta[i]));
                stage_idx[n_active] = i;
                stage_val[n_active] = act >= 0.0 ? 1 : -1;
                ++n_active;
            }
            /* synchronous commit (_kernels.py:154-155) */
            for (int64_t a = 0; a < n_active; ++a) spins[stage_idx[a]] = stage_val[a];
        }
        /* per-cycle energy then cut, same order as _kernels.py:157-165 */
        double e = 0.0;
        for (int64_t i = 0; i < n; ++i) e -= h[i] * (double)spins[i];
        for (int64_t t = 0; t < mm; ++t)
            e -= me_w[t] * (double)spins[me_i[t]] * (double)spins[me_j[t]];
        int64_t cut = 0;
        for (int64_t t = 0; t < gm; ++t)
            if (spins[ge_i[t]] != spins[ge_j[t]]) cut += ge_w[t];
        trace_i0[c] = i0;
        trace_energy[c] = e;
        trace_cut[c] = cut;
        if (cut > best) best = cut;
        if (c < cycles - 1) i0 = i0 / beta;
    }
    *best_cut = best;
    free(stage_idx);
    free(stage_val);
    return 0;
}

/* ------------------------------------------------------------------ batch */
/*
 * Many independent trials over a pool of pthreads -- the restated form of
 * engine.run_trials' ThreadPoolExecutor fan-out (engine.py:118-123).  Per
 * trial t the profile rows are lam[t*n..], delta[t*n..], period[t*n..]
 * (profile_stride = n) or shared (profile_stride = 0).  Outputs are laid out
 * [T][...] contiguously.
 */
int orc_anneal_batch_rng(int64_t T, int nthreads, int64_t n, const int64_t *indptr,
                         const int64_t *indices, const double *values, const double *h, int64_t mm,
                         const int64_t *me_i, const int64_t *me_j, const double *me_w, int64_t gm,
                         const int64_t *ge_i, const int64_t *ge_j, const int64_t *ge_w,
                         const double *lam, const double *delta, const int64_t *period,
                         int64_t profile_stride, double i0_min, double beta, int64_t cycles,
                         int64_t t_res, int algo, int64_t alpha, double p_stall,
                         const uint64_t *keys, int rng, uint64_t seed, int64_t first_trial,
                         int8_t *spins, double *inputs, double *hist, int64_t *counts,
                         double *trace_i0, double *trace_energy, int64_t *trace_cut,
                         int64_t *best_cut);

typedef struct {
    int64_t n, mm, gm;
    const int64_t *indptr, *indices, *me_i, *me_j, *ge_i, *ge_j, *ge_w, *period;
    const double *values, *h, *me_w, *lam, *delta;
    int64_t profile_stride;
    double i0_min, beta, p_stall;
    int64_t cycles, t_res, alpha;
    int algo;
    const uint64_t *keys;
    int rng;
    uint64_t seed;
    int64_t first_trial;
    int64_t T;
    int8_t *spins;
    double *inputs, *hist, *trace_i0, *trace_energy;
    int64_t *counts, *trace_cut, *best_cut;
    int64_t next;
    pthread_mutex_t lock;
    int status;
} orc_batch_t;

static void *orc_worker(void *arg) {
    orc_batch_t *b = (orc_batch_t *)arg;
    for (;;) {
        pthread_mutex_lock(&b->lock);
        int64_t t = b->next++;
        pthread_mutex_unlock(&b->lock);
        if (t >= b->T) break;
        int64_t n = b->n, ps = b->profile_stride, C = b->cycles;
        int rc = orc_anneal_rng(n, b->indptr, b->indices, b->values, b->h, b->mm, b->me_i, b->me_j,
                            b->me_w, b->gm, b->ge_i, b->ge_j, b->ge_w, b->lam + t * ps,
                            b->delta + t * ps, b->period + t * ps, b->i0_min, b->beta, C,
                            b->t_res, b->algo, b->alpha, b->p_stall, b->keys[t], b->rng,
                            b->seed, b->first_trial + t,
                            b->spins + t * n, b->inputs + t * n, b->hist + t * n * b->alpha,
                            b->counts + t * n, b->trace_i0 + t * C, b->trace_energy + t * C,
                            b->trace_cut + t * C, b->best_cut + t);
        if (rc != 0) b->status = rc;
    }
    return NULL;
}

int orc_anneal_batch(int64_t T, int nthreads, int64_t n, const int64_t *indptr,
                     const int64_t *indices, const double *values, const double *h, int64_t mm,
                     const int64_t *me_i, const int64_t *me_j, const double *me_w, int64_t gm,
                     const int64_t *ge_i, const int64_t *ge_j, const int64_t *ge_w,
                     const double *lam, const double *delta, const int64_t *period,
                     int64_t profile_stride, double i0_min, double beta, int64_t cycles,
                     int64_t t_res, int algo, int64_t alpha, double p_stall,
                     const uint64_t *keys, int8_t *spins, double *inputs, double *hist,
                     int64_t *counts, double *trace_i0, double *trace_energy,
                     int64_t *trace_cut, int64_t *best_cut) {
    return orc_anneal_batch_rng(T, nthreads, n, indptr, indices, values, h, mm, me_i, me_j, me_w,
                                gm, ge_i, ge_j, ge_w, lam, delta, period, profile_stride, i0_min,
                                beta, cycles, t_res, algo, alpha, p_stall, keys, 0, 0, 0, spins,
                                inputs, hist, counts, trace_i0, trace_energy, trace_cut, best_cut);
}

/* orc_anneal_batch with a choice of stream; trial t is global trial first_trial + t. */
int orc_anneal_batch_rng(int64_t T, int nthreads, int64_t n, const int64_t *indptr,
                         const int64_t *indices, const double *values, const double *h, int64_t mm,
                         const int64_t *me_i, const int64_t *me_j, const double *me_w, int64_t gm,
                         const int64_t *ge_i, const int64_t *ge_j, const int64_t *ge_w,
                         const double *lam, const double *delta, const int64_t *period,
                         int64_t profile_stride, double i0_min, double beta, int64_t cycles,
                         int64_t t_res, int algo, int64_t alpha, double p_stall,
                         const uint64_t *keys, int rng, uint64_t seed, int64_t first_trial,
                         int8_t *spins, double *inputs, double *hist, int64_t *counts,
                         double *trace_i0, double *trace_energy, int64_t *trace_cut,
                         int64_t *best_cut) {
    orc_batch_t b;
    memset(&b, 0, sizeof b);
    b.rng = rng; b.seed = seed; b.first_trial = first_trial;
    b.n = n; b.mm = mm; b.gm = gm;
    b.indptr = indptr; b.indices = indices; b.values = values; b.h = h;
    b.me_i = me_i; b.me_j = me_j; b.me_w = me_w;
    b.ge_i = ge_i; b.ge_j = ge_j; b.ge_w = ge_w;
    b.lam = lam; b.delta = delta; b.period = period; b.profile_stride = profile_stride;
    b.i0_min = i0_min; b.beta = beta; b.p_stall = p_stall;
    b.cycles = cycles; b.t_res = t_res; b.alpha = alpha; b.algo = algo;
    b.keys = keys; b.T = T;
    b.spins = spins; b.inputs = inputs; b.hist = hist; b.counts = counts;
    b.trace_i0 = trace_i0; b.trace_energy = trace_energy; b.trace_cut = trace_cut;
    b.best_cut = best_cut;
    pthread_mutex_init(&b.lock, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 1024) nthreads = 1024;
    pthread_t tid[1024];
    int started = 0;
    for (int k = 1; k < nthreads; ++k)
        if (pthread_create(&tid[started], NULL, orc_worker, &b) == 0) ++started;
    orc_worker(&b);
    for (int k = 0; k < started; ++k) pthread_join(tid[k], NULL);
    pthread_mutex_destroy(&b.lock);
    return b.status;
}
