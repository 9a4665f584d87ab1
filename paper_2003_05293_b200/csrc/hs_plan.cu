// hs_plan.cu -- host runtime + C ABI (include/holospots_b200.h).
//
// A plan owns one pupil's geometry on one device: the storage-order pixel
// list, the block-sorted dense list used by full-range passes, and a cache
// of block-sorted compressed-window lists (one per window offset of the
// CS-WGS schedule, solvers.py:212-222).  Solves are recorded once per
// (algorithm, iterations, subset, batch, spots, flags) into a CUDA graph
// and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/holospots_b200.h"
#include "hs_kernels.cuh"

using namespace hs;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                              \
    do {                                                                            \
        cudaError_t e_ = (expr);                                                    \
        if (e_ != cudaSuccess)                                                      \
            return fail(HS_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));  \
    } while (0)

constexpr int kBlock = 64;  // spatial sort block (pixels) for pixel lists

struct DevList {
    int32_t *rc = nullptr;
    float *amp = nullptr;
    int32_t *dst = nullptr;
    int64_t count = 0;
};

template <typename T>
int dalloc(T **p, size_t count)
{
    *p = nullptr;
    if (count == 0) return HS_OK;
    cudaError_t e = cudaMalloc((void **)p, count * sizeof(T));
    if (e != cudaSuccess)
        return fail(HS_ECUDA, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
    return HS_OK;
}

template <typename T>
void dfree(T *&p)
{
    if (p) cudaFree(p);
    p = nullptr;
}

struct Config {
    int G, L, nl, np;
};

Config pick_config(int n)
{
    Config c{};
    if (n <= 16) { c.G = 1; c.L = 16; }
    else if (n <= 32) { c.G = 2; c.L = 16; }
    else if (n <= 64) { c.G = 4; c.L = 16; }
    else if (n <= 128) { c.G = 8; c.L = 16; }
    else if (n <= 256) { c.G = 16; c.L = 16; }
    else if (n <= 512) { c.G = 32; c.L = 16; }
    else { c.G = 32; c.L = 32; }
    c.nl = (n + c.G - 1) / c.G;
    c.np = c.G * c.nl;
    return c;
}

typedef void (*PassFn)(PassArgs);

template <int G, int L>
PassFn pass_fn(int mode)
{
    switch (mode) {
    case PM_BWD | PM_WRITE: return hs_pass_kernel<G, L, PM_BWD | PM_WRITE>;
    case PM_FWD: return hs_pass_kernel<G, L, PM_FWD>;
    case PM_BWD | PM_FWD: return hs_pass_kernel<G, L, PM_BWD | PM_FWD>;
    case PM_BWD | PM_FWD | PM_WRITE: return hs_pass_kernel<G, L, PM_BWD | PM_FWD | PM_WRITE>;
    default: return nullptr;
    }
}

PassFn select_pass(const Config &c, int mode)
{
    if (c.L == 32) return pass_fn<32, 32>(mode);
    switch (c.G) {
    case 1: return pass_fn<1, 16>(mode);
    case 2: return pass_fn<2, 16>(mode);
    case 4: return pass_fn<4, 16>(mode);
    case 8: return pass_fn<8, 16>(mode);
    case 16: return pass_fn<16, 16>(mode);
    default: return pass_fn<32, 16>(mode);
    }
}

}  // namespace

struct hs_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    int side = 0;
    int64_t m = 0;
    double c1 = 0, c2 = 0, sum_amp = 0;
    std::vector<int32_t> h_rows, h_cols;
    std::vector<float> h_amp;
    double *d_axis = nullptr;
    DevList storage;  // storage order, dst = nullptr
    DevList dense;    // block-sorted, dst = storage index
    std::map<std::pair<int64_t, int64_t>, DevList> windows;

    // spot batch
    int batch = 0, n = 0, cap_batch = 0, cap_np = 0;
    Config cfg{};
    bool tables_valid = false;
    double *d_x = nullptr, *d_y = nullptr, *d_z = nullptr, *d_a0 = nullptr;
    double *d_theta = nullptr, *d_amp_in = nullptr;
    float2 *d_gx = nullptr, *d_gy = nullptr;
    double *d_w = nullptr;
    float2 *d_coef = nullptr;
    float2 *d_part = nullptr;
    int64_t part_stride = 0;
    int32_t *d_status = nullptr, *d_degen = nullptr, *d_qstatus = nullptr;
    double *d_fields = nullptr, *d_e = nullptr, *d_u = nullptr, *d_inten = nullptr, *d_rel = nullptr;
    double *d_phase = nullptr;   // [cap_batch][m] solver output / API scratch
    double *d_trace_w = nullptr, *d_trace_m = nullptr;
    int64_t trace_cap = 0;

    // last solve
    int last_alg = -1, last_iters = 0, last_flags = 0;
    int64_t last_launches = 0;

    // graph cache
    std::map<std::tuple<int, int, int64_t, int, int, int>, cudaGraphExec_t> graphs;

    int launches = 0;  // counter while recording
};

namespace {

void sort_list(const hs_plan *p, std::vector<int64_t> &idx)
{
    const int nb = (p->side + kBlock - 1) / kBlock;
    std::vector<std::pair<int64_t, int64_t>> keyed(idx.size());
    for (size_t i = 0; i < idx.size(); ++i) {
        const int64_t s = idx[i];
        const int64_t r = p->h_rows[s], c = p->h_cols[s];
        const int64_t key = ((r / kBlock) * nb + c / kBlock) * (int64_t)(kBlock * kBlock) +
                            (r % kBlock) * kBlock + (c % kBlock);
        keyed[i] = {key, s};
    }
    std::sort(keyed.begin(), keyed.end());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = keyed[i].second;
}

int upload_list(const hs_plan *p, const std::vector<int64_t> &idx, bool with_dst, DevList *out)
{
    const int64_t cnt = (int64_t)idx.size();
    std::vector<int32_t> rc(cnt), dst(with_dst ? cnt : 0);
    std::vector<float> amp(cnt);
    for (int64_t i = 0; i < cnt; ++i) {
        const int64_t s = idx[i];
        rc[i] = (p->h_rows[s] << 16) | p->h_cols[s];
        amp[i] = p->h_amp[s];
        if (with_dst) dst[i] = (int32_t)s;
    }
    int rcode;
    if ((rcode = dalloc(&out->rc, cnt)) || (rcode = dalloc(&out->amp, cnt))) return rcode;
    if (with_dst && (rcode = dalloc(&out->dst, cnt))) return rcode;
    out->count = cnt;
    if (cnt) {
        CUDA_TRY(cudaMemcpy(out->rc, rc.data(), cnt * sizeof(int32_t), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(out->amp, amp.data(), cnt * sizeof(float), cudaMemcpyHostToDevice));
        if (with_dst)
            CUDA_TRY(cudaMemcpy(out->dst, dst.data(), cnt * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    return HS_OK;
}

void free_list(DevList &l)
{
    dfree(l.rc);
    dfree(l.amp);
    dfree(l.dst);
    l.count = 0;
}

int get_window(hs_plan *p, int64_t start, int64_t count, const DevList **out)
{
    if (start == 0 && count == p->m) {
        *out = &p->dense;
        return HS_OK;
    }
    auto key = std::make_pair(start, count);
    auto it = p->windows.find(key);
    if (it == p->windows.end()) {
        std::vector<int64_t> idx(count);
        for (int64_t i = 0; i < count; ++i) idx[i] = start + i;
        sort_list(p, idx);
        DevList l;
        int rc = upload_list(p, idx, false, &l);
        if (rc) return rc;
        it = p->windows.emplace(key, l).first;
    }
    *out = &it->second;
    return HS_OK;
}

void free_graphs(hs_plan *p)
{
    for (auto &kv : p->graphs) cudaGraphExecDestroy(kv.second);
    p->graphs.clear();
}

void free_batch(hs_plan *p)
{
    dfree(p->d_x); dfree(p->d_y); dfree(p->d_z); dfree(p->d_a0);
    dfree(p->d_theta); dfree(p->d_amp_in);
    dfree(p->d_gx); dfree(p->d_gy); dfree(p->d_w); dfree(p->d_coef); dfree(p->d_part);
    dfree(p->d_status); dfree(p->d_degen); dfree(p->d_qstatus);
    dfree(p->d_fields); dfree(p->d_e); dfree(p->d_u); dfree(p->d_inten); dfree(p->d_rel);
    dfree(p->d_phase);
    dfree(p->d_trace_w); dfree(p->d_trace_m);
    p->cap_batch = p->cap_np = 0;
    p->trace_cap = 0;
    free_graphs(p);
}

int ensure_batch(hs_plan *p, int batch, int n)
{
    const Config cfg = pick_config(n);
    if (batch <= p->cap_batch && cfg.np <= p->cap_np && n <= p->cap_np) return HS_OK;
    free_batch(p);
    const int B = batch;
    const int np = cfg.np;
    const size_t bn = (size_t)B * np;
    p->part_stride = (int64_t)(kTargetChunks + 8) * np;
    int rc;
    if ((rc = dalloc(&p->d_x, bn)) || (rc = dalloc(&p->d_y, bn)) || (rc = dalloc(&p->d_z, bn)) ||
        (rc = dalloc(&p->d_a0, bn)) || (rc = dalloc(&p->d_theta, bn)) ||
        (rc = dalloc(&p->d_amp_in, bn)) ||
        (rc = dalloc(&p->d_gx, (size_t)B * p->side * np)) ||
        (rc = dalloc(&p->d_gy, (size_t)B * p->side * np)) || (rc = dalloc(&p->d_w, bn)) ||
        (rc = dalloc(&p->d_coef, bn)) || (rc = dalloc(&p->d_part, (size_t)B * p->part_stride)) ||
        (rc = dalloc(&p->d_status, B)) || (rc = dalloc(&p->d_degen, B)) ||
        (rc = dalloc(&p->d_qstatus, B)) || (rc = dalloc(&p->d_fields, bn * 2)) ||
        (rc = dalloc(&p->d_e, B)) || (rc = dalloc(&p->d_u, B)) || (rc = dalloc(&p->d_inten, bn)) ||
        (rc = dalloc(&p->d_rel, bn)) || (rc = dalloc(&p->d_phase, (size_t)B * p->m))) {
        free_batch(p);
        return rc;
    }
    p->cap_batch = B;
    p->cap_np = np;
    return HS_OK;
}

int ensure_trace(hs_plan *p, int iters)
{
    const int64_t need = (int64_t)p->batch * std::max(iters, 1) * p->n;
    if (need <= p->trace_cap) return HS_OK;
    dfree(p->d_trace_w);
    dfree(p->d_trace_m);
    int rc;
    if ((rc = dalloc(&p->d_trace_w, need)) || (rc = dalloc(&p->d_trace_m, need))) return rc;
    p->trace_cap = need;
    free_graphs(p);  // graphs bake the trace pointers
    return HS_OK;
}

// ---- launch helpers (record into the current stream / capture) ----------

struct PassGeom {
    int32_t chunk_len;
    int32_t nchunks;
};

PassGeom pass_geom(int64_t count, int G)
{
    const int nslots = kThreads / G;
    int64_t per = (count + kTargetChunks - 1) / kTargetChunks;
    per = ((per + nslots - 1) / nslots) * nslots;
    if (per < nslots) per = nslots;
    PassGeom g;
    g.chunk_len = (int32_t)per;
    g.nchunks = (int32_t)((count + per - 1) / per);
    return g;
}

int launch_tables(hs_plan *p)
{
    dim3 grid(p->side, p->batch);
    hs_tables_kernel<<<grid, 128, 0, p->stream>>>(p->side, p->cfg.np, p->n, p->d_axis, p->c1, p->c2,
                                                  p->d_x, p->d_y, p->d_z, p->d_gx, p->d_gy);
    p->launches++;
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}

// Launch one pass over `list` (+offset) for all patterns; returns nchunks.
int launch_pass(hs_plan *p, int mode, const int32_t *rc, const float *amp, const int32_t *dst,
                int64_t idx_base, int64_t count, const double *phase_in, double *phase_out,
                int64_t phase_stride, int32_t *nchunks_out)
{
    const Config &c = p->cfg;
    PassGeom geo = pass_geom(count, c.G);
    *nchunks_out = geo.nchunks;
    if (count == 0) return HS_OK;
    PassArgs a;
    a.rc = rc;
    a.amp = amp;
    a.dst = dst;
    a.idx_base = idx_base;
    a.count = count;
    a.chunk_len = geo.chunk_len;
    a.side = p->side;
    a.np = c.np;
    a.tab_stride = (int64_t)p->side * c.np;
    a.gx = p->d_gx;
    a.gy = p->d_gy;
    a.coef = p->d_coef;
    a.phase_in = phase_in;
    a.phase_out = phase_out;
    a.phase_stride = phase_stride;
    a.partials = p->d_part;
    a.part_stride = p->part_stride;
    a.status = p->d_status;
    PassFn fn = select_pass(c, mode);
    const size_t smem = (mode & PM_FWD) ? (size_t)(kThreads / c.G) * c.np * sizeof(float2) : 0;
    dim3 grid(geo.nchunks, p->batch);
    fn<<<grid, kThreads, smem, p->stream>>>(a);
    p->launches++;
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}

UpdArgs upd_args(hs_plan *p, int mode, int nchunks)
{
    UpdArgs u;
    memset(&u, 0, sizeof u);
    u.mode = mode;
    u.n = p->n;
    u.np = p->cfg.np;
    u.nchunks = nchunks;
    u.partials = p->d_part;
    u.part_stride = p->part_stride;
    u.amp_in = p->d_amp_in;
    u.theta_in = p->d_theta;
    u.a0 = p->d_a0;
    u.w = p->d_w;
    u.coef = p->d_coef;
    u.trace_w = p->d_trace_w;
    u.trace_m = p->d_trace_m;
    u.status = p->d_status;
    u.degen = p->d_degen;
    u.qstatus = p->d_qstatus;
    u.fields = p->d_fields;
    u.inv_norm = 1.0 / (p->sum_amp * p->sum_amp);
    u.e = p->d_e;
    u.u = p->d_u;
    u.inten = p->d_inten;
    u.rel = p->d_rel;
    return u;
}

int launch_update(hs_plan *p, const UpdArgs &u)
{
    hs_update_kernel<<<p->batch, kUpdThreads, 0, p->stream>>>(u);
    p->launches++;
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}

int reset_status(hs_plan *p)
{
    CUDA_TRY(cudaMemsetAsync(p->d_status, 0, sizeof(int32_t) * p->batch, p->stream));
    CUDA_TRY(cudaMemsetAsync(p->d_degen, 0, sizeof(int32_t) * p->batch, p->stream));
    CUDA_TRY(cudaMemsetAsync(p->d_qstatus, 0, sizeof(int32_t) * p->batch, p->stream));
    return HS_OK;
}

int ensure_tables(hs_plan *p)
{
    if (p->tables_valid) return HS_OK;
    int rc = launch_tables(p);
    if (rc) return rc;
    p->tables_valid = true;
    return HS_OK;
}

// The solve schedule (solvers.py:192-235), fused:
//   pass_0 = superpose(coef_0) + forward over read_1
//   for j = 1..I: update_j (forward fields of pass_{j-1} -> coef_j);
//                 pass_j = superpose(coef_j) over write_j + forward over write_j
//                 (= read_{j+1}); the last pass writes the phase and yields
//                 the full-range fields of quality_report.
int record_solve(hs_plan *p, int alg, int iters, int64_t subset, int flags)
{
    int rc;
    const bool want_fields = (flags & HS_WANT_FIELDS) != 0;
    if ((rc = reset_status(p))) return rc;
    if ((rc = launch_tables(p))) return rc;
    UpdArgs seed = upd_args(p, UPD_SEED, 0);
    seed.amp_in = p->d_a0;
    if ((rc = launch_update(p, seed))) return rc;
    int32_t nch = 0;
    const int64_t m = p->m;
    if (alg == HS_ALG_RS) {
        const int mode = want_fields ? (PM_BWD | PM_FWD | PM_WRITE) : (PM_BWD | PM_WRITE);
        if ((rc = launch_pass(p, mode, p->dense.rc, p->dense.amp, p->dense.dst, 0, m, nullptr,
                              p->d_phase, m, &nch)))
            return rc;
        if (want_fields && (rc = launch_update(p, upd_args(p, UPD_FINAL, nch)))) return rc;
        return HS_OK;
    }
    const int cs = (subset < m) ? std::max(0, iters - 2) : 0;
    const int64_t half = std::max<int64_t>(1, subset / 2);
    // window written by iteration j (1-based), j <= cs
    auto window_of = [&](int j, const DevList **l) -> int {
        const int64_t off = ((int64_t)(j - 1) * half) % (m - subset + 1);
        return get_window(p, off, subset, l);
    };
    const DevList *lst = nullptr;
    if (cs > 0) {
        if ((rc = get_window(p, 0, subset, &lst))) return rc;
    } else {
        lst = &p->dense;
    }
    if ((rc = launch_pass(p, PM_BWD | PM_FWD, lst->rc, lst->amp, nullptr, 0, lst->count, nullptr,
                          nullptr, 0, &nch)))
        return rc;
    for (int j = 1; j <= iters; ++j) {
        UpdArgs u = upd_args(p, UPD_STEP, nch);
        u.iter = j - 1;
        u.iters = iters;
        if ((rc = launch_update(p, u))) return rc;
        const bool last = (j == iters);
        if (j <= cs) {
            if ((rc = window_of(j, &lst))) return rc;
        } else {
            lst = &p->dense;
        }
        if (last) {
            const int mode = want_fields ? (PM_BWD | PM_FWD | PM_WRITE) : (PM_BWD | PM_WRITE);
            if ((rc = launch_pass(p, mode, lst->rc, lst->amp, lst->dst, 0, lst->count, nullptr,
                                  p->d_phase, m, &nch)))
                return rc;
            if (want_fields && (rc = launch_update(p, upd_args(p, UPD_FINAL, nch)))) return rc;
        } else {
            if ((rc = launch_pass(p, PM_BWD | PM_FWD, lst->rc, lst->amp, nullptr, 0, lst->count,
                                  nullptr, nullptr, 0, &nch)))
                return rc;
        }
    }
    return HS_OK;
}

int check_device(hs_plan *p)
{
    CUDA_TRY(cudaSetDevice(p->device));
    return HS_OK;
}

int sync_and_check(hs_plan *p)
{
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}

}  // namespace

// ============================================================ C ABI ========
extern "C" {

const char *hs_last_error(void) { return g_err.c_str(); }

int hs_device_count(int *count)
{
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    *count = n;
    return HS_OK;
}

int hs_max_spots(void) { return 1024; }

int hs_plan_create(int device, int side, int64_t m, const int64_t *rows, const int64_t *cols,
                   const double *amplitude, const double *axis, double prism, double lens,
                   double sum_amplitude, hs_plan **out)
{
    *out = nullptr;
    if (side < 2 || side > 65535) return fail(HS_EINVAL, "side_px %d outside 2..65535", side);
    if (m < 1 || m > (int64_t)side * side) return fail(HS_EINVAL, "pixel count %lld invalid", (long long)m);
    if (m > INT32_MAX) return fail(HS_EINVAL, "pixel count too large");
    std::unique_ptr<hs_plan> p(new hs_plan);
    p->device = device;
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->side = side;
    p->m = m;
    p->c1 = prism;
    p->c2 = lens;
    p->sum_amp = sum_amplitude;
    p->h_rows.resize(m);
    p->h_cols.resize(m);
    p->h_amp.resize(m);
    for (int64_t i = 0; i < m; ++i) {
        if (rows[i] < 0 || rows[i] >= side || cols[i] < 0 || cols[i] >= side)
            return fail(HS_EINVAL, "pixel %lld outside the grid", (long long)i);
        p->h_rows[i] = (int32_t)rows[i];
        p->h_cols[i] = (int32_t)cols[i];
        p->h_amp[i] = (float)amplitude[i];
    }
    int rc;
    if ((rc = dalloc(&p->d_axis, side))) return rc;
    CUDA_TRY(cudaMemcpy(p->d_axis, axis, sizeof(double) * side, cudaMemcpyHostToDevice));
    std::vector<int64_t> idx(m);
    for (int64_t i = 0; i < m; ++i) idx[i] = i;
    if ((rc = upload_list(p.get(), idx, false, &p->storage))) return rc;
    sort_list(p.get(), idx);
    if ((rc = upload_list(p.get(), idx, true, &p->dense))) return rc;
    // 64 KB dynamic shared memory for the widest pass variant.
    const int modes[4] = {PM_BWD | PM_WRITE, PM_FWD, PM_BWD | PM_FWD, PM_BWD | PM_FWD | PM_WRITE};
    for (int mode : modes) {
        Config c{32, 32, 32, 1024};
        CUDA_TRY(cudaFuncSetAttribute(select_pass(c, mode), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      65536));
    }
    *out = p.release();
    return HS_OK;
}

void hs_plan_destroy(hs_plan *p)
{
    if (!p) return;
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->stream);
    free_batch(p);
    free_list(p->storage);
    free_list(p->dense);
    for (auto &kv : p->windows) free_list(kv.second);
    dfree(p->d_axis);
    cudaStreamDestroy(p->stream);
    delete p;
}

int hs_set_spots(hs_plan *p, int batch, int n, const double *x, const double *y, const double *z,
                 const double *a0)
{
    if (batch < 1) return fail(HS_EINVAL, "batch must be >= 1");
    if (n < 1 || n > hs_max_spots()) return fail(HS_EINVAL, "spot count %d outside 1..%d", n, hs_max_spots());
    int rc;
    if ((rc = check_device(p))) return rc;
    if ((rc = ensure_batch(p, batch, n))) return rc;
    if (p->batch != batch || p->n != n) free_graphs(p);
    p->batch = batch;
    p->n = n;
    p->cfg = pick_config(n);
    const size_t bytes = sizeof(double) * (size_t)batch * n;
    CUDA_TRY(cudaMemcpyAsync(p->d_x, x, bytes, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->d_y, y, bytes, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->d_z, z, bytes, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->d_a0, a0, bytes, cudaMemcpyHostToDevice, p->stream));
    p->tables_valid = false;
    return HS_OK;
}

int hs_superpose(hs_plan *p, const double *amplitude, const double *theta, int64_t start, int64_t stop,
                 double *out)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    if (start < 0 || start > stop || stop > p->m)
        return fail(HS_EINVAL, "pixel range (%lld, %lld) outside 0..%lld", (long long)start,
                    (long long)stop, (long long)p->m);
    int rc;
    if ((rc = check_device(p)) || (rc = ensure_tables(p)) || (rc = reset_status(p))) return rc;
    const size_t bytes = sizeof(double) * p->n;
    CUDA_TRY(cudaMemcpyAsync(p->d_amp_in, amplitude, bytes, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->d_theta, theta, bytes, cudaMemcpyHostToDevice, p->stream));
    const int saved = p->batch;
    p->batch = 1;
    UpdArgs seed = upd_args(p, UPD_SEED, 0);
    seed.w = nullptr;
    rc = launch_update(p, seed);
    int32_t nch;
    if (!rc)
        rc = launch_pass(p, PM_BWD | PM_WRITE, p->storage.rc + start, p->storage.amp + start, nullptr, 0,
                         stop - start, nullptr, p->d_phase, 0, &nch);
    p->batch = saved;
    if (rc) return rc;
    if (stop > start)
        CUDA_TRY(cudaMemcpyAsync(out, p->d_phase, sizeof(double) * (stop - start), cudaMemcpyDeviceToHost,
                                 p->stream));
    return sync_and_check(p);
}

static int forward_common(hs_plan *p, const double *phase, int64_t start, int64_t stop, int mode)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    if (start < 0 || start > stop || stop > p->m)
        return fail(HS_EINVAL, "pixel range (%lld, %lld) outside 0..%lld", (long long)start,
                    (long long)stop, (long long)p->m);
    int rc;
    if ((rc = check_device(p)) || (rc = ensure_tables(p)) || (rc = reset_status(p))) return rc;
    CUDA_TRY(cudaMemcpyAsync(p->d_phase, phase, sizeof(double) * p->m, cudaMemcpyHostToDevice, p->stream));
    const int saved = p->batch;
    p->batch = 1;
    int32_t nch = 0;
    if (stop > start) {
        rc = launch_pass(p, PM_FWD, p->storage.rc + start, p->storage.amp + start, nullptr, start,
                         stop - start, p->d_phase, nullptr, 0, &nch);
    } else {
        // empty range: zero fields (kernels.py:234-235) via a zero partial
        cudaMemsetAsync(p->d_part, 0, sizeof(float2) * p->cfg.np, p->stream);
        nch = 1;
    }
    if (!rc) rc = launch_update(p, upd_args(p, mode, nch));
    p->batch = saved;
    return rc;
}

int hs_forward(hs_plan *p, const double *phase, int64_t start, int64_t stop, double *fields)
{
    int rc = forward_common(p, phase, start, stop, UPD_FIELDS);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(fields, p->d_fields, sizeof(double) * 2 * p->n, cudaMemcpyDeviceToHost,
                             p->stream));
    return sync_and_check(p);
}

int hs_quality(hs_plan *p, const double *phase, double *e, double *u, double *intensities,
               double *relative, double *fields)
{
    if (!(p->sum_amp > 0.0)) return fail(HS_EZEROILLUM, "pupil carries no illumination");
    int rc = forward_common(p, phase, 0, p->m, UPD_FINAL);
    if (rc) return rc;
    int32_t qs = 0;
    CUDA_TRY(cudaMemcpyAsync(e, p->d_e, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaMemcpyAsync(u, p->d_u, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaMemcpyAsync(&qs, p->d_qstatus, sizeof(int32_t), cudaMemcpyDeviceToHost, p->stream));
    if (intensities)
        CUDA_TRY(cudaMemcpyAsync(intensities, p->d_inten, sizeof(double) * p->n, cudaMemcpyDeviceToHost,
                                 p->stream));
    if (relative)
        CUDA_TRY(cudaMemcpyAsync(relative, p->d_rel, sizeof(double) * p->n, cudaMemcpyDeviceToHost,
                                 p->stream));
    if (fields)
        CUDA_TRY(cudaMemcpyAsync(fields, p->d_fields, sizeof(double) * 2 * p->n, cudaMemcpyDeviceToHost,
                                 p->stream));
    if ((rc = sync_and_check(p))) return rc;
    if (qs) return fail(HS_EUNDEFINED, "all spot intensities are zero");
    return HS_OK;
}

int hs_solve_async(hs_plan *p, int alg, int iters, int64_t subset, const double *theta0, int flags)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    if (alg != HS_ALG_RS && alg != HS_ALG_WGS && alg != HS_ALG_CSWGS)
        return fail(HS_EINVAL, "unknown algorithm %d", alg);
    if (alg == HS_ALG_RS) {
        iters = 0;
        subset = p->m;
    } else {
        if (iters < 1) return fail(HS_EINVAL, "iterations must be >= 1");
        if (alg == HS_ALG_CSWGS && iters < 2) return fail(HS_EINVAL, "cswgs needs iterations >= 2");
        if (alg == HS_ALG_WGS) subset = p->m;
        if (subset < 1 || subset > p->m) return fail(HS_EINVAL, "subset size %lld outside 1..M", (long long)subset);
    }
    if ((flags & HS_WANT_FIELDS) && !(p->sum_amp > 0.0))
        return fail(HS_EZEROILLUM, "pupil carries no illumination");
    int rc;
    if ((rc = check_device(p))) return rc;
    if ((rc = ensure_trace(p, iters))) return rc;
    // windows are built (host sort + upload) outside capture
    if (alg != HS_ALG_RS && subset < p->m && iters > 2) {
        const int64_t half = std::max<int64_t>(1, subset / 2);
        for (int j = 1; j <= iters - 2; ++j) {
            const DevList *l;
            if ((rc = get_window(p, ((int64_t)(j - 1) * half) % (p->m - subset + 1), subset, &l))) return rc;
        }
    }
    const size_t bytes = sizeof(double) * (size_t)p->batch * p->n;
    CUDA_TRY(cudaMemcpyAsync(p->d_theta, theta0, bytes, cudaMemcpyHostToDevice, p->stream));
    auto key = std::make_tuple(alg, iters, subset, flags, p->batch, p->n);
    auto it = p->graphs.find(key);
    if (it == p->graphs.end()) {
        cudaGraph_t graph;
        p->launches = 0;
        CUDA_TRY(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
        rc = record_solve(p, alg, iters, subset, flags);
        cudaError_t ce = cudaStreamEndCapture(p->stream, &graph);
        if (rc) return rc;
        if (ce != cudaSuccess) return fail(HS_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
        cudaGraphExec_t exec;
        ce = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return fail(HS_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
        it = p->graphs.emplace(key, exec).first;
        p->last_launches = p->launches;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, p->stream));
    p->tables_valid = true;
    p->last_alg = alg;
    p->last_iters = iters;
    p->last_flags = flags;
    {
        // launches recorded for this key: recount cheaply from the schedule
        int64_t l = 3;  // tables + seed + first pass
        if (alg != HS_ALG_RS) l += 2LL * iters;
        if (flags & HS_WANT_FIELDS) l += 1;
        p->last_launches = l;
    }
    return HS_OK;
}

int hs_solve(hs_plan *p, int alg, int iters, int64_t subset, const double *theta0, int flags)
{
    int rc = hs_solve_async(p, alg, iters, subset, theta0, flags);
    if (rc) return rc;
    return sync_and_check(p);
}

int hs_sync(hs_plan *p)
{
    int rc;
    if ((rc = check_device(p))) return rc;
    return sync_and_check(p);
}

int hs_get_status(hs_plan *p, int32_t *status, int32_t *degenerate)
{
    int rc;
    if ((rc = check_device(p))) return rc;
    if (status)
        CUDA_TRY(cudaMemcpyAsync(status, p->d_status, sizeof(int32_t) * p->batch, cudaMemcpyDeviceToHost,
                                 p->stream));
    if (degenerate)
        CUDA_TRY(cudaMemcpyAsync(degenerate, p->d_degen, sizeof(int32_t) * p->batch,
                                 cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

int hs_get_trace(hs_plan *p, double *weights, double *mags)
{
    int rc;
    if ((rc = check_device(p))) return rc;
    const size_t cnt = (size_t)p->batch * p->last_iters * p->n;
    if (cnt) {
        if (weights)
            CUDA_TRY(cudaMemcpyAsync(weights, p->d_trace_w, sizeof(double) * cnt, cudaMemcpyDeviceToHost,
                                     p->stream));
        if (mags)
            CUDA_TRY(cudaMemcpyAsync(mags, p->d_trace_m, sizeof(double) * cnt, cudaMemcpyDeviceToHost,
                                     p->stream));
    }
    return sync_and_check(p);
}

int hs_get_phase(hs_plan *p, int first, int count, double *phase)
{
    if (first < 0 || count < 0 || first + count > p->batch) return fail(HS_EINVAL, "pattern range invalid");
    int rc;
    if ((rc = check_device(p))) return rc;
    if (count)
        CUDA_TRY(cudaMemcpyAsync(phase, p->d_phase + (size_t)first * p->m, sizeof(double) * count * p->m,
                                 cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

int hs_get_quality(hs_plan *p, double *e, double *u, double *intensities, double *relative, double *fields)
{
    if (!(p->last_flags & HS_WANT_FIELDS)) return fail(HS_EINVAL, "last solve did not compute fields");
    int rc;
    if ((rc = check_device(p))) return rc;
    const size_t B = p->batch, bn = (size_t)p->batch * p->n;
    if (e) CUDA_TRY(cudaMemcpyAsync(e, p->d_e, sizeof(double) * B, cudaMemcpyDeviceToHost, p->stream));
    if (u) CUDA_TRY(cudaMemcpyAsync(u, p->d_u, sizeof(double) * B, cudaMemcpyDeviceToHost, p->stream));
    if (intensities)
        CUDA_TRY(cudaMemcpyAsync(intensities, p->d_inten, sizeof(double) * bn, cudaMemcpyDeviceToHost, p->stream));
    if (relative)
        CUDA_TRY(cudaMemcpyAsync(relative, p->d_rel, sizeof(double) * bn, cudaMemcpyDeviceToHost, p->stream));
    if (fields)
        CUDA_TRY(cudaMemcpyAsync(fields, p->d_fields, sizeof(double) * 2 * bn, cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

int hs_solve_host(hs_plan *p, int alg, int iters, int64_t subset, int batch, int n, const double *x,
                  const double *y, const double *z, const double *a0, const double *theta0, double *phase,
                  double *e, double *u)
{
    int rc;
    if ((rc = hs_set_spots(p, batch, n, x, y, z, a0))) return rc;
    if ((rc = hs_solve_async(p, alg, iters, subset, theta0, HS_WANT_FIELDS))) return rc;
    if (phase)
        CUDA_TRY(cudaMemcpyAsync(phase, p->d_phase, sizeof(double) * (size_t)batch * p->m,
                                 cudaMemcpyDeviceToHost, p->stream));
    if (e) CUDA_TRY(cudaMemcpyAsync(e, p->d_e, sizeof(double) * batch, cudaMemcpyDeviceToHost, p->stream));
    if (u) CUDA_TRY(cudaMemcpyAsync(u, p->d_u, sizeof(double) * batch, cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

void *hs_plan_stream(hs_plan *p) { return (void *)p->stream; }

int hs_last_launch_count(hs_plan *p, int64_t *launches)
{
    *launches = p->last_launches;
    return HS_OK;
}

int hs_time_kernel(hs_plan *p, int which, int64_t subset, int reps, double *ms_per_launch,
                   double *pairs_per_launch)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    if (reps < 1) return fail(HS_EINVAL, "reps must be >= 1");
    int rc;
    if ((rc = check_device(p)) || (rc = ensure_tables(p))) return rc;
    const DevList *l = &p->dense;
    if (which == 1) {
        if (subset < 1 || subset > p->m) return fail(HS_EINVAL, "subset invalid");
        if ((rc = get_window(p, 0, subset, &l))) return rc;
    }
    if ((rc = ensure_trace(p, 1))) return rc;
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    int32_t nch = 0;
    auto once = [&]() -> int {
        if (which == 2) {
            UpdArgs u = upd_args(p, UPD_STEP, nch);
            u.iter = 0;
            u.iters = 1;
            return launch_update(p, u);
        }
        return launch_pass(p, PM_BWD | PM_FWD, l->rc, l->amp, nullptr, 0, l->count, nullptr, nullptr, 0, &nch);
    };
    if (which == 2) {
        // make the update meaningful: produce partials once
        if ((rc = launch_pass(p, PM_BWD | PM_FWD, l->rc, l->amp, nullptr, 0, l->count, nullptr, nullptr, 0,
                              &nch)))
            return rc;
    }
    if ((rc = reset_status(p)) || (rc = once()) || (rc = reset_status(p))) return rc;
    CUDA_TRY(cudaEventRecord(e0, p->stream));
    for (int r = 0; r < reps; ++r) {
        if ((rc = once())) return rc;
    }
    CUDA_TRY(cudaEventRecord(e1, p->stream));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_per_launch = ms / reps;
    *pairs_per_launch = (which == 2) ? 0.0 : (double)l->count * p->n * p->batch;
    return reset_status(p);
}

void *hs_host_alloc(int64_t bytes)
{
    void *ptr = nullptr;
    if (cudaHostAlloc(&ptr, (size_t)bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return ptr;
}

void hs_host_free(void *ptr)
{
    if (ptr) cudaFreeHost(ptr);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// FP32 FMA-pipe peak microbenchmark (roofline denominator: MEASURED_PEAKS.json
// carries only HBM and bf16-tensor figures).  8 independent FFMA chains per
// thread, 148 x 8 CTAs of 256 threads.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(256) hs_ffma_kernel(float *out, int iters, float a, float b)
{
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    float x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 1.2345f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

extern "C" int hs_fma_peak(int device, double *tflops)
{
    CUDA_TRY(cudaSetDevice(device));
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float *out = nullptr;
    CUDA_TRY(cudaMalloc(&out, sizeof(float) * blocks * threads));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    hs_ffma_kernel<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);  // warm
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CUDA_TRY(cudaEventRecord(e0));
        hs_ffma_kernel<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
        CUDA_TRY(cudaEventRecord(e1));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    *tflops = flops / (best * 1e-3) / 1e12;
    return HS_OK;
}
