// debug.cu -- debug kernels (hash, Philox, prefilter, tanh), the trace CSV formatter
// and host exports of the hash and threshold helpers
#include "runtime.h"

extern "C" {

int pbsa_debug_stream_u64(int device, int64_t count, const uint64_t *key, const uint64_t *tag,
                          const uint64_t *a, const uint64_t *b, uint64_t *out) {
    return guarded([&] {
        if (count < 0) fail(PBSA_EINVAL, "negative count");
        if (count == 0) return;
        DeviceGuard dg(device);
        DevBuf<uint64_t> dk, dt, da, db, dout;
        dk.upload(key, count, 0);
        dt.upload(tag, count, 0);
        da.upload(a, count, 0);
        db.upload(b, count, 0);
        dout.alloc(count);
        pbsa::debug_stream<<<grid_for(count, 256), 256>>>(count, dk.p, dt.p, da.p, db.p, dout.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, dout.p, count * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    });
}

int pbsa_debug_philox(int device, int64_t count, const uint32_t *ctr, const uint32_t *key,
                      uint32_t *out) {
    return guarded([&] {
        if (count < 0 || (count > 0 && (!ctr || !key || !out))) fail(PBSA_EINVAL, "bad arguments");
        if (count == 0) return;
        DeviceGuard dg(device);
        DevBuf<uint32_t> dc, dk, dout;
        dc.upload(ctr, 4 * count, 0);
        dk.upload(key, 2 * count, 0);
        dout.alloc((size_t)(4 * count));
        pbsa::debug_philox<<<grid_for(count, 256), 256>>>(count, dc.p, dk.p, dout.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, dout.p, sizeof(uint32_t) * 4 * count, cudaMemcpyDeviceToHost));
    });
}

int pbsa_debug_var_prefilter(int device, int64_t count, const double *lam, const double *delta,
                             const double *i0, const int *raw, const uint32_t *zh, uint32_t *out) {
    return guarded([&] {
        if (count < 0 || (count > 0 && (!lam || !delta || !i0 || !raw || !zh || !out)))
            fail(PBSA_EINVAL, "bad arguments");
        if (count == 0) return;
        DeviceGuard dg(device);
        DevBuf<double> dl, dd, di;
        DevBuf<int> dr;
        DevBuf<uint32_t> dz, dout;
        dl.upload(lam, count, 0);
        dd.upload(delta, count, 0);
        di.upload(i0, count, 0);
        dr.upload(raw, count, 0);
        dz.upload(zh, count, 0);
        dout.alloc(count);
        pbsa::debug_var_prefilter<<<grid_for(count, 256), 256>>>(count, dl.p, dd.p, di.p, dr.p, dz.p, dout.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, dout.p, sizeof(uint32_t) * count, cudaMemcpyDeviceToHost));
    });
}

int pbsa_debug_tanh(int device, int64_t count, const double *x, double *out) {
    return guarded([&] {
        if (count < 0) fail(PBSA_EINVAL, "negative count");
        if (count == 0) return;
        DeviceGuard dg(device);
        DevBuf<double> dx, dout;
        dx.upload(x, count, 0);
        dout.alloc(count);
        pbsa::debug_tanh<<<grid_for(count, 256), 256>>>(count, dx.p, dout.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, dout.p, count * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

// ------------------------------------------------------- trace CSV text
// Host-side formatter behind paper_2601_14476_b200.traces:
// the rows "trial,cycle,i0,energy,cut\n" of the reference CLI's trace file
// (cli.py:163-168), for integral energies, written by all host threads.
namespace {
inline int dec_len(uint64_t x) {
    int n = 1;
    while (x >= 10) { x /= 10; ++n; }
    return n;
}
inline int int_len(int64_t v) {
    return v < 0 ? 1 + dec_len((uint64_t)0 - (uint64_t)v) : dec_len((uint64_t)v);
}
inline char *put_int(char *p, int64_t v) {
    uint64_t x = (uint64_t)v;
    if (v < 0) { *p++ = '-'; x = (uint64_t)0 - x; }
    char tmp[24];
    int n = 0;
    do { tmp[n++] = (char)('0' + x % 10); x /= 10; } while (x);
    while (n) *p++ = tmp[--n];
    return p;
}
}  // namespace

int pbsa_format_trace_csv(int64_t T, int64_t C, const char *i0_text, const int64_t *i0_off,
                          const int64_t *energy, const int64_t *cut, char *out, int64_t out_cap,
                          int64_t *out_len) {
    return guarded([&] {
        if (T < 0 || C < 0 || (T * C > 0 && (!i0_text || !i0_off || !energy || !out)) || !out_len)
            fail(PBSA_EINVAL, "bad arguments");
        std::vector<int64_t> tlen(T + 1, 0);
        parallel_for(T, 16, [&](int64_t t0, int64_t t1) {
            for (int64_t t = t0; t < t1; ++t) {
                int64_t len = 0;
                const int tl = int_len(t);
                for (int64_t c = 0; c < C; ++c) {
                    // "t,c,i0,E.0,cut\n": four commas, ".0" and the newline
                    len += tl + int_len(c) + (i0_off[c + 1] - i0_off[c]) + int_len(energy[t * C + c]) +
                           (cut ? int_len(cut[t * C + c]) : 0) + 7;
                }
                tlen[t + 1] = len;
            }
        });
        for (int64_t t = 0; t < T; ++t) tlen[t + 1] += tlen[t];
        *out_len = tlen[T];
        if (tlen[T] > out_cap) fail(PBSA_EINVAL, "output buffer too small (%lld bytes needed)", (long long)tlen[T]);
        parallel_for(T, 16, [&](int64_t t0, int64_t t1) {
            for (int64_t t = t0; t < t1; ++t) {
                char *p = out + tlen[t];
                for (int64_t c = 0; c < C; ++c) {
                    p = put_int(p, t);
                    *p++ = ',';
                    p = put_int(p, c);
                    *p++ = ',';
                    const int64_t a = i0_off[c], b = i0_off[c + 1];
                    std::memcpy(p, i0_text + a, (size_t)(b - a));
                    p += b - a;
                    *p++ = ',';
                    p = put_int(p, energy[t * C + c]);
                    *p++ = '.';
                    *p++ = '0';
                    *p++ = ',';
                    if (cut) p = put_int(p, cut[t * C + c]);
                    *p++ = '\n';
                }
            }
        });
    });
}

double pbsa_libm_tanh_host(double x) { return pb_libm_tanh(x); }

uint64_t pbsa_threshold_host(double t) { return threshold_h64(t); }

uint64_t pbsa_threshold_native_host(double t) { return threshold_native(t); }

void pbsa_philox_host(const uint32_t *ctr, const uint32_t *key, uint32_t *out) {
    uint32_t o[4];
    pbsa::philox4x32_10(ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1], o);
    for (int k = 0; k < 4; ++k) out[k] = o[k];
}

}  // extern "C"
