// runtime.h -- internal header of the host runtime (not part of the C ABI):
// the plan object, error plumbing, device buffers, host hash helpers and the
// kernel selectors shared by the runtime translation units
//   plan.cu     plan creation (layout choice, uploads, tables)
//   launch.cu   the anneal enqueue (captured into a graph or launched directly)
//   abi.cu      plan entry points of include/pbsa.h and the output download
//   oneshot.cu  the one-shot batch calls, their plan cache and device fan-out
//   debug.cu    debug kernels, trace CSV formatter and host hash exports
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pbsa.h"
#include "aux_kernels.cuh"
#include "dispatch.h"

extern char **environ;

namespace pbsa_rt {

inline thread_local std::string g_last_error;
// set while pbsa_anneal_loop_batch builds its single-use plan: such plans skip
// word phasing, whose graph (phases x chains x cycles nodes) costs more to
// instantiate than a single run saves
inline thread_local bool g_oneshot = false;
// set while a cacheable one-shot call builds its plan: the plan keeps the
// benchmark's launch structure (word phases, chains) captured into one graph,
// with each phase's output formatting and copies to the caller's (page-locked)
// buffers captured into it too, so a later call of the same shape replays it
inline thread_local bool g_cached_oneshot = false;
// bytes the calling thread's last one-shot call moved (pbsa_last_call_bytes)
inline thread_local int64_t g_call_h2d = 0, g_call_d2h = 0;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Error(code, buf);
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            fail(e_ == cudaErrorMemoryAllocation ? PBSA_ENOMEM : PBSA_ECUDA, "%s: %s (%s:%d)", \
                 #call, cudaGetErrorString(e_), __FILE__, __LINE__);                    \
    } while (0)

template <typename F>
inline int guarded(F &&f) {
    try {
        f();
        return PBSA_OK;
    } catch (const Error &e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        g_last_error = "host allocation failed";
        return PBSA_ENOMEM;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return PBSA_EINVAL;
    }
}

// -------------------------------------------------------------- host hash
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
inline uint64_t hmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D4A04C32684F87ULL;
    return z ^ (z >> 31);
}
inline uint64_t habsorb(uint64_t h, uint64_t w) { return hmix64((h + kGamma) ^ w); }

// Smallest integer U with U * 2^-52 - 1 + t >= 0, i.e. ceil((1 - t) * 2^52),
// computed exactly from t's binary representation (t in [-1, 1]).
inline uint64_t threshold_u53(double t) {
    if (t == 0.0) return 1ULL << 52;
    int e;
    const double f = std::frexp(t, &e);                  // t = f 2^e, |f| in [0.5, 1)
    const int64_t M = (int64_t)std::ldexp(f, 53);        // exact 53-bit integer
    const int sh = e - 1;                                // t * 2^52 = M * 2^sh
    const int64_t two52 = 1LL << 52;
    if (sh >= 0) return (uint64_t)(two52 - (M << sh));
    const int k = -sh;
    if (M > 0) {
        if (k >= 63) return (uint64_t)two52;             // ceil(2^52 - tiny)
        return (uint64_t)(two52 - (M >> k));
    }
    const int64_t A = -M;
    if (k >= 63) return (uint64_t)two52 + 1;
    const int64_t q = (A >> k) + ((A & ((1LL << k) - 1)) ? 1 : 0);
    return (uint64_t)(two52 + q);
}

// Native mode (philox.cuh): +1 iff (2X + 1) 2^-32 - 1 + t >= 0, i.e.
// (2X + 1) 2^20 >= U = ceil((1 - t) 2^52); the smallest such 32-bit X,
// 2^32 meaning "never".
inline uint64_t threshold_native(double t) {
    const uint64_t u = threshold_u53(t);
    if (u <= (1ULL << 20)) return 0;
    return (u - (1ULL << 20) + (1ULL << 21) - 1) >> 21;
}

inline uint64_t threshold_h64(double t) {
    const uint64_t u = threshold_u53(t);
    if (u >= (1ULL << 53)) return ~0ULL;  // never +1
    return u << 11;
}

inline int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Stream-ordered device buffers from the device's default memory pool (its
// release threshold is raised once per device, so repeated one-shot calls
// reuse memory instead of paying cudaMalloc/cudaFree each time).
inline thread_local cudaStream_t g_alloc_stream = nullptr;

struct AllocStream {
    cudaStream_t prev;
    explicit AllocStream(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
    ~AllocStream() { g_alloc_stream = prev; }
};

template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    size_t bytes_up = 0;  // host->device bytes of the last upload
    cudaStream_t st = nullptr;
    void alloc(size_t count) {
        release();
        n = count;
        st = g_alloc_stream;
        if (count) CK(cudaMallocAsync(reinterpret_cast<void **>(&p), count * sizeof(T), st));
    }
    void upload(const T *src, size_t count, cudaStream_t s) {
        alloc(count);
        bytes_up = count * sizeof(T);
        if (count) CK(cudaMemcpyAsync(p, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T> &v, cudaStream_t s) { upload(v.data(), v.size(), s); }
    // new contents for an existing buffer of the same size (its device address,
    // captured into a cached graph, stays)
    void overwrite(const std::vector<T> &v, cudaStream_t s) {
        if (v.size() != n) fail(PBSA_EINVAL, "cached plan buffer size changed");
        bytes_up = v.size() * sizeof(T);
        if (n) CK(cudaMemcpyAsync(p, v.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void release() {
        drop();
        bytes_up = 0;
    }
    void drop() {  // free the memory early; keep the upload byte count for pbsa_plan_bytes
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
};

inline void raise_pool_threshold(int device) {
    static std::mutex mu;
    static std::set<int> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(device)) return;
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    done.insert(device);
}

// Fill a large host array with several threads (output buffers of a full
// 4096-trial G81 download are ~0.7 GB each).
template <typename T>
inline void parallel_fill(T *dst, size_t count, T value) {
    const size_t bytes = count * sizeof(T);
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (bytes < (32u << 20) || nt == 1) {
        std::fill(dst, dst + count, value);
        return;
    }
    std::vector<std::thread> pool;
    const size_t per = (count + nt - 1) / nt;
    for (unsigned k = 0; k < nt; ++k) {
        const size_t lo = k * per, hi = std::min(count, lo + per);
        if (lo >= hi) break;
        pool.emplace_back([=] { std::fill(dst + lo, dst + hi, value); });
    }
    for (auto &t : pool) t.join();
}

// Run f(lo, hi) over [0, count) split across host threads (large layouts only).
template <typename F>
inline void parallel_for(int64_t count, int64_t min_per_thread, F &&f) {
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    nt = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nt, count / std::max<int64_t>(1, min_per_thread)));
    if (nt == 1) {
        f((int64_t)0, count);
        return;
    }
    std::vector<std::thread> pool;
    const int64_t per = (count + nt - 1) / nt;
    for (unsigned k = 0; k < nt; ++k) {
        const int64_t lo = k * per, hi = std::min(count, lo + per);
        if (lo >= hi) break;
        pool.emplace_back([&f, lo, hi] { f(lo, hi); });
    }
    for (auto &t : pool) t.join();
}

inline int64_t grid_for(int64_t work, int threads) { return (work + threads - 1) / threads; }

}  // namespace

using namespace pbsa_rt;

struct StreamHolder {
    cudaStream_t s = nullptr;
    ~StreamHolder() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

struct PbsaHostOut {  // caller's output buffers of a pipelined one-shot call
    int8_t *spins;
    double *inputs, *trace_energy;
    int64_t *trace_cut, *best;
};

struct pbsa_plan {
    // declared first so it is destroyed last, after every buffer has been
    // released onto it
    StreamHolder stream_holder;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaEvent_t ev_start = nullptr, ev_sweep0 = nullptr, ev_sweep1 = nullptr, ev_end = nullptr;
    cudaEvent_t ev_fork = nullptr;
    std::vector<cudaEvent_t> ev_join;
    std::vector<cudaStream_t> chain_streams;  // packed path: extra concurrent word groups
    bool ran = false;

    // problem
    int64_t n = 0, T = 0, Tp = 0, W = 0, cycles = 0, t_res = 0, alpha = 1, nnz = 0;
    int algo = 0;
    double p_stall = 0.5;
    int path = 0;
    bool has_graph = false;
    bool int_energy = true;
    bool tapsa_hist_from_raw = false;  // TAPSA alpha=1 routed to the packed path
    bool tapsa_packed = false;         // TAPSA alpha>=2 on the packed path (bit-sliced ring)
    // one-shot pipelined mode: the run is not captured into a graph; word
    // phases run one after another and each phase's outputs are formatted and
    // copied to the caller's host buffers on out_stream while the next computes
    bool pipelined = false;
    bool capturing_outputs = false;    // a cached one-shot plan: phase outputs inside the graph
    bool direct = false;               // one-shot: launched directly, no graph (instantiation costs more)
    std::vector<std::pair<cudaGraphNode_t, int>> out_nodes;  // its D2H copy nodes and output index
    std::vector<size_t> out_node_off;  // destination byte offset of each node in its output
    std::vector<size_t> out_node_bytes;
    std::vector<const void *> out_node_src;
    void *out_bound[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // caller buffers the graph writes
    // cached one-shot plans ship the last raw fields as int16 (trial-major) to a
    // page-locked staging buffer and widen them to the caller's fp64 inputs on
    // host threads as each word phase lands (a host node per phase signals it)
    DevBuf<int16_t> o_raw16;           // [T][n] device
    int16_t *h_raw = nullptr;          // [T][n] page-locked staging
    struct PhaseCb {
        pbsa_plan *P;
        int k;
    };
    std::vector<PhaseCb> cb_args;
    std::vector<std::pair<int64_t, int64_t>> phase_trials;  // [t0, t1) per phase
    std::mutex cb_mu;
    std::condition_variable cb_cv;
    int cb_done = 0;
    cudaStream_t out_stream = nullptr;
    std::vector<cudaEvent_t> ev_phase;
    PbsaHostOut hout{};
    int64_t mm_ = 0, gm_ = 0;          // model / graph edge counts (direct enqueue)
    DevBuf<int8_t> o_spins;
    DevBuf<double> o_inputs;
    bool native = false;               // PBSA_RNG_PHILOX: Philox draws (philox.cuh)
    bool reg4 = false;                 // packed path: every degree is 4 (gather_counts_reg4)
    uint64_t nseed = 0;                // Philox key
    int64_t first_trial = 0;           // global index of trial 0 (Philox trial groups)
    bool spsa_packed = false;          // SPSA p>0 on the packed path (per-p-bit drive index)
    DevBuf<uint32_t> sidx;             // [W][32][n] drive index per p-bit
    bool sidx_full = true;             // store every index (PBSA_SIDX_FULL=0: fresh ones only)
    DevBuf<uint32_t> thr_hi;           // [cycles][K] high words of the thresholds
    DevBuf<uint2> kfs;                 // [Tp] (F, C) of absorb(key, TAG_STALL) + GAMMA
    DevBuf<uint64_t> kstg;             // [Tp] absorb(key, TAG_STALL) + GAMMA
    DevBuf<double> i0_dev;             // [cycles]
    uint64_t p_stall64 = 0;
    DevBuf<uint32_t> ring;             // [W][alpha][L][n]
    int64_t total_w = 0;
    std::vector<double> i0;
    std::vector<uint32_t> active_counts;  // general path: sub-steps with any update
    int64_t launches = 0, sweep_launches = 0;
    int64_t updates_per_run = 0;

    // packed path
    int L = 1, dmax = 0, K = 1;
    int warps_per_word = 1, chunks = 1, packed_blocks = 1;
    bool cta_flush = false;           // packed_sweep: one cut flush per block (warps_per_word % warps == 0)
    DevBuf<uint32_t> p_spins[2], rowptr, adj;  // adj: 32-bit CSR entries (n > 32768)
    DevBuf<uint16_t> adj16;                     // 16-bit CSR entries (n <= 32768)
    DevBuf<uint32_t> order;                     // [chunks * 32] degree-sorted processing order, or empty
    DevBuf<uint64_t> thr, krg;
    DevBuf<uint2> kfc, acache;
    bool use_cache = false;
    bool use_pdl = true;  // PBSA_PDL=0 disables programmatic dependent launch
    int64_t phase_words = 1;
    DevBuf<unsigned long long> pacc;  // [(C+1)][Tp]
    DevBuf<int16_t> raw_last;         // [n][Tp]
    // packed VAR mode: per-p-bit variability profile under the plain rule
    bool var_mode = false, var_uniform = true;
    DevBuf<float2> prof;               // [Tp][n] {fl32(lam), fl32(lam * delta)} (no timing spread)
    DevBuf<__half2> prof16;            // [W][n][32] {fl16(lam), fl16(lam * delta)} (timing spread)
    DevBuf<double> lam64, del64;       // [Tp][n]
    DevBuf<double> inp_var;            // [Tp][n] last i0 * raw of every p-bit
    DevBuf<uint32_t> pplanes;          // [W][nplanes][n]
    DevBuf<uint8_t> vdivs;             // divisor lists of all sub-steps
    int nplanes = 0;
    int64_t pmax = 0;
    float var_margin = 1.0f;
    std::vector<uint8_t> pcl;          // [T][n] clamped periods (timing spread only)
    // timing spread on the launched path: period buckets (packed_sweep_bucket)
    bool bucket = false;
    int nclass = 0;                    // distinct clamped periods present
    int max_ndiv = 0;                  // most classes firing in one sub-step
    DevBuf<uint8_t> bdivs;             // like vdivs, as class indices
    DevBuf<uint4> brec;                // [W][chunks][1024] slot records (slot, fp16 profile pair, hash cache)
    DevBuf<uint16_t> boff;             // [W][chunks][nclass + 1] class starts
    DevBuf<uint8_t> blut;              // [256] clamped period -> class
    DevBuf<uint8_t> bcper;             // [nclass] class -> clamped period
    // packed launch sequence (one entry per sweep launch, the last one cut-only)
    struct PLaunch {
        uint32_t count;
        int64_t cycle;
        int do_cut, ndiv;
        int64_t div_off;
        bool update, inp;
    };
    std::vector<PLaunch> plaunch;
    // resident mode: one cluster per word anneals all cycles in one launch
    bool resident = false, res_timing = false, res_prof_smem = false, res_split = false;
    bool res_tapsa = false;
    int res_cs = 1, res_threads = 256;
    size_t res_smem = 0;
    DevBuf<pbsa::RLaunch> rlaunch;     // resident timing: the sub-step list

    // general path
    DevBuf<int8_t> g_spins[2];
    DevBuf<uint32_t> col, me_i, me_j, ge_i, ge_j;
    DevBuf<double> val, h, me_w, lam, delta, inputs, hist, e_f64;
    DevBuf<int64_t> me_wi, h_int, ge_w;
    DevBuf<int32_t> period, counts;
    DevBuf<uint64_t> kr, kst;
    DevBuf<unsigned long long> cut_acc, e_acc, dj_acc;  // [C][Tp]
    DevBuf<int32_t> ge_w32, me_w32;
    int64_t sum_j = 0;
    bool graph_is_model = false;
    int shared_profile = 0;
    bool has_lam = false, has_delta = false, has_period = false;
    // active-list mode (integer-valued models): per-sub-step lists of firing p-bits
    struct ALaunch {
        uint32_t count;
        int64_t cycle, desc_off;
        int ndesc, total;
    };
    bool active_mode = false;
    std::vector<ALaunch> alaunch;
    DevBuf<uint32_t> alist, st_g;
    DevBuf<int8_t> st_v;
    DevBuf<int4> adesc;
    DevBuf<int32_t> vali, hi32, hist_i, a_counts;  // hist_i: [alpha][Np], list order
    DevBuf<double> a_inputs;                        // [Np], list order
    DevBuf<uint64_t> athr;  // [cycles][Kt] thresholds (lam = 1, delta = 0, plain rule), or empty
    int tshift = 0, rawmin = 0, Kt = 0;
    // fast active mode (plain rule): folded draw, fp32 profile, flips only
    bool fast = false;
    DevBuf<float2> aprof;                 // [Np] list order or [n] shared
    DevBuf<uint32_t> flips, nflips;       // [max firing] / [launches]
    int64_t apmax = 1;                    // largest clamped period
    std::vector<int32_t> apcl;            // [T][n] clamped periods (host counts)
    std::vector<uint64_t> kr_host;        // [Tp] absorb(key, TAG_R)
    // cached one-shot plans: host copies of the key-independent uploads (the
    // cache key fixes their content; each call uploads them again)
    std::vector<uint32_t> h_rowptr, h_adj32;
    std::vector<uint16_t> h_adj16;
    std::vector<uint64_t> h_thr;
    uint32_t tmask = 0;

    DevBuf<uint64_t> kspin;
    // outputs
    DevBuf<int64_t> trace_cut, best;
    DevBuf<double> trace_energy;
    int final_parity = 0;  // which spin buffer holds the final state

    cudaGraph_t graph = nullptr;       // kept for a cached plan (its copy nodes are updated)
    ~pbsa_plan() {
        if (h_raw) {
            if (out_stream) cudaStreamSynchronize(out_stream);
            if (stream) cudaStreamSynchronize(stream);
            cudaFreeHost(h_raw);
        }
        // drain every stream first: after an error in a pipelined one-shot call
        // the output stream may still be formatting and copying phase outputs
        // into the caller's host buffers, reading buffers released below
        if (out_stream) cudaStreamSynchronize(out_stream);
        for (cudaStream_t cs : chain_streams) cudaStreamSynchronize(cs);
        if (stream) cudaStreamSynchronize(stream);
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        if (graph) cudaGraphDestroy(graph);
        for (cudaEvent_t e : {ev_start, ev_sweep0, ev_sweep1, ev_end, ev_fork})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_join) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_phase) cudaEventDestroy(e);
        if (out_stream) cudaStreamDestroy(out_stream);
        for (cudaStream_t cs : chain_streams) cudaStreamDestroy(cs);
    }
};

namespace pbsa_rt {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CK(cudaGetDevice(&prev));
        CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

inline bool is_integral(double x) { return std::isfinite(x) && x == std::nearbyint(x) && std::fabs(x) < 2147483647.0; }

template <typename K>
inline void set_packed_smem(K kernel, size_t bytes) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

using pbsa_dispatch::PackedKernel;
using pbsa_dispatch::ResidentKernel;
using pbsa_dispatch::ResidentTimingKernel;

// The sweep kernels live in the per-L translation units (dispatch.h).
inline PackedKernel packed_kernel_for(int L, bool update, bool cached, bool tapsa = false,
                               bool spsa = false, int var = 0, bool native = false) {
#define PBSA_PK(l) packed_kernel<l>(update, cached, tapsa, spsa, var, native)
    switch (L) {
        case 1: return pbsa_dispatch::PBSA_PK(1);
        case 2: return pbsa_dispatch::PBSA_PK(2);
        case 3: return pbsa_dispatch::PBSA_PK(3);
        case 4: return pbsa_dispatch::PBSA_PK(4);
        case 5: return pbsa_dispatch::PBSA_PK(5);
        case 6: return pbsa_dispatch::PBSA_PK(6);
        case 7: return pbsa_dispatch::PBSA_PK(7);
        default: fail(PBSA_EINVAL, "packed path supports degree <= 127");
    }
#undef PBSA_PK
}

inline PackedKernel bucket_kernel_for(int L, bool native) {
    switch (L) {
        case 1: return pbsa_dispatch::bucket_kernel<1>(native);
        case 2: return pbsa_dispatch::bucket_kernel<2>(native);
        case 3: return pbsa_dispatch::bucket_kernel<3>(native);
        case 4: return pbsa_dispatch::bucket_kernel<4>(native);
        case 5: return pbsa_dispatch::bucket_kernel<5>(native);
        case 6: return pbsa_dispatch::bucket_kernel<6>(native);
        case 7: return pbsa_dispatch::bucket_kernel<7>(native);
        default: fail(PBSA_EINVAL, "packed variability path supports degree <= 127");
    }
}

inline ResidentTimingKernel resident_timing_for(int L, bool native = false) {
    switch (L) {
        case 1: return pbsa_dispatch::resident_timing_kernel<1>(native);
        case 2: return pbsa_dispatch::resident_timing_kernel<2>(native);
        case 3: return pbsa_dispatch::resident_timing_kernel<3>(native);
        case 4: return pbsa_dispatch::resident_timing_kernel<4>(native);
        case 5: return pbsa_dispatch::resident_timing_kernel<5>(native);
        case 6: return pbsa_dispatch::resident_timing_kernel<6>(native);
        case 7: return pbsa_dispatch::resident_timing_kernel<7>(native);
        default: fail(PBSA_EINVAL, "resident sweep supports degree <= 127");
    }
}

inline ResidentKernel resident_kernel_for(int L, bool cached, bool varu = false, bool native = false,
                                   bool tapsa = false) {
#define PBSA_RK(l) resident_kernel<l>(cached, varu, native, tapsa)
    switch (L) {
        case 1: return pbsa_dispatch::PBSA_RK(1);
        case 2: return pbsa_dispatch::PBSA_RK(2);
        case 3: return pbsa_dispatch::PBSA_RK(3);
        case 4: return pbsa_dispatch::PBSA_RK(4);
        case 5: return pbsa_dispatch::PBSA_RK(5);
        case 6: return pbsa_dispatch::PBSA_RK(6);
        case 7: return pbsa_dispatch::PBSA_RK(7);
        default: fail(PBSA_EINVAL, "resident sweep supports degree <= 127");
    }
#undef PBSA_RK
}

template <int L>
inline void launch_hist_from_ring(const uint32_t *ring, const uint32_t *rowptr, int n, int T, int alpha,
                           int written, double *out, cudaStream_t st) {
    pbsa::hist_from_ring<L><<<grid_for((int64_t)n * T, 256), 256, 0, st>>>(ring, rowptr, n, T, alpha,
                                                                          written, out);
}
}  // namespace pbsa_rt

// ------------------------------------------------ cross-unit entry points
namespace pbsa_rt {
int64_t choose_phases(int64_t chunks, int64_t W, int64_t resident_warps, size_t l2_budget, bool *balance);
void setup_active(pbsa_plan &P, int64_t n, const int64_t *indptr, const int64_t *indices,
                  const double *values, const double *hv, const double *lam, const double *delta,
                  const int64_t *period, int64_t pstride, int64_t trials, int64_t cycles,
                  int64_t t_res, int algo, int64_t alpha, double p_stall);
void host_trial_keys(const uint64_t *keys, int64_t trials, int64_t Tp, std::vector<uint64_t> &kspin,
                     std::vector<uint64_t> &kr, std::vector<uint64_t> &kst);
void host_packed_consts(const std::vector<uint64_t> &kr, std::vector<uint64_t> &krg, std::vector<uint2> &kfc);
std::vector<uint64_t> host_plain_thresholds(const pbsa_plan &P);
void host_csr(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
              std::vector<uint32_t> &rowptr, std::vector<uint32_t> &adj32, std::vector<uint16_t> &adj16);
void create_plan(pbsa_plan &P, int device, int64_t n, const int64_t *indptr,
                 const int64_t *indices, const double *values, const double *hv, int64_t mm,
                 const int64_t *mei, const int64_t *mej, const double *mew, int64_t gm,
                 const int64_t *gei, const int64_t *gej, const int64_t *gew, const double *lam,
                 const double *delta, const int64_t *period, int64_t pstride, double i0_min,
                 double beta, int64_t cycles, int64_t t_res, int algo, int64_t alpha,
                 double p_stall, int64_t trials, const uint64_t *keys, int rng_mode,
                 uint64_t rng_seed, int64_t first_trial, const double *native_sig = nullptr);
cudaError_t record_sweep_event(const pbsa_plan &P, cudaEvent_t ev, cudaStream_t st);
void CUDART_CB phase_landed(void *arg);
void enqueue_phase_outputs(pbsa_plan &P, int64_t w0, int64_t w1, int parity, int k);
void enqueue_run(pbsa_plan &P, int64_t mm, int64_t gm);
void launch_run(pbsa_plan &P);
int plan_create_impl(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                     const double *values, const double *h, int64_t mm, const int64_t *me_i,
                     const int64_t *me_j, const double *me_w, int64_t gm, const int64_t *ge_i,
                     const int64_t *ge_j, const int64_t *ge_w, const double *lam,
                     const double *delta, const int64_t *period, int64_t profile_stride,
                     double i0_min, double beta, int64_t cycles, int64_t t_res, int algo,
                     int64_t alpha, double p_stall, int64_t trials, const uint64_t *keys,
                     int rng_mode, uint64_t rng_seed, int64_t first_trial, const double *native_sig,
                     pbsa_plan **out);
void host_constant_outputs(pbsa_plan *P, double *hist, int64_t *counts, double *trace_i0);
void download_impl(pbsa_plan *P, int8_t *spins, double *inputs, double *hist, int64_t *counts,
                   double *trace_i0, double *trace_energy, int64_t *trace_cut, int64_t *best_cut,
                   bool consts_done);
uint64_t hash_bytes(const void *p, size_t bytes, uint64_t h);
bool pinned_or_null(const void *p);
pbsa_plan *plan_cache_take(const std::vector<uint64_t> &key);
void plan_cache_put(std::vector<uint64_t> key, pbsa_plan *P);
void graph_outputs(const pbsa_plan &P, const PbsaHostOut &h, void *(&ptr)[5], size_t (&bytes)[5]);
void capture_with_outputs(pbsa_plan &P, const PbsaHostOut &hout);
void bind_outputs(pbsa_plan &P, const PbsaHostOut &hout);
void refresh_inputs(pbsa_plan &P, int64_t n, const int64_t *indptr, const int64_t *indices,
                    const double *values, const uint64_t *keys);
}  // namespace pbsa_rt

