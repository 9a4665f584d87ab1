// hs_kernels.cuh -- sm_100a device kernels of the CS-WGS hot path.
//
//   hs_tables_kernel  per-pattern column/row unit phasors gx, gy
//                     (reference _build_tables, holospots/kernels.py:78-96)
//   hs_pass_kernel    fused pixel pass over a pixel list: back-propagation
//                     S_p = sum_n coef_n gx[c_p,n] gy[r_p,n] -> arg (kernels.py:99-119)
//                     and/or forward projection E_n += b_p gx gy with
//                     b_p = A_p e^{-i arg S_p} (kernels.py:122-144), one
//                     deterministic partial per (pattern, chunk)
//   hs_update_kernel  fixed-order fp64 fold of the chunk partials + the
//                     weight / theta update (solvers.py:96-163) or the
//                     e / u epilogue (metrics.py:33-79)
//
// Numerics: phasor arguments are formed in fp64 in the
// reference's operation order (no FMA contraction) and rounded to fp32
// phasors; the pixel loops run in fp32 on the FMA pipe; every reduction
// across pixels is a fixed-shape tree whose shape depends only on the list
// length, never on scheduling, so results are bitwise run-to-run stable and
// independent of batch size.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hs {

constexpr int kThreads = 256;        // pass-kernel CTA size
constexpr int kTargetChunks = 296;   // 2 x 148 SMs: chunks per pattern and pass
constexpr int kUpdThreads = 1024;
constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 6.283185307179586;

enum PassMode : int { PM_BWD = 1, PM_FWD = 2, PM_WRITE = 4 };

struct PassArgs {
    const int32_t *rc;        // packed (row << 16) | col per list entry
    const float *amp;         // illumination amplitude per entry
    const int32_t *dst;       // phase index per entry (nullptr: i + idx_base)
    int64_t idx_base;
    int64_t count;            // list length
    int32_t chunk_len;        // entries per CTA (multiple of the slot count)
    int32_t side;
    int32_t np;               // padded spot count (G * spots-per-lane)
    int64_t tab_stride;       // side * np
    const float2 *gx, *gy;    // [B][side][np]
    const float2 *coef;       // [B][np]   superposition coefficients
    const double *phase_in;   // [B][phase_stride] (PM_FWD without PM_BWD)
    double *phase_out;        // [B][phase_stride] (PM_WRITE)
    int64_t phase_stride;
    float2 *partials;         // [B][part_stride]: [chunk][np]
    int64_t part_stride;
    const int32_t *status;    // [B] nonzero -> pattern already failed, skip
};

// ---------------------------------------------------------------------------
// Tables: gx[b][j][n] = exp(i (c1 x_n a_j + c2 z_n a_j^2)), gy likewise with
// y_n.  The argument is formed with explicit round-to-nearest fp64 ops in the
// reference order ((c1*x)*v + (c2*z)*v2), so it equals numba's argument bit
// for bit; sincos runs in fp64 and the phasor is rounded once to fp32.
// ---------------------------------------------------------------------------
__global__ void hs_tables_kernel(int side, int np, int n, const double *__restrict__ axis,
                                 double c1, double c2, const double *__restrict__ x,
                                 const double *__restrict__ y, const double *__restrict__ z,
                                 float2 *__restrict__ gx, float2 *__restrict__ gy)
{
    const int j = blockIdx.x;
    const int b = blockIdx.y;
    const double v = axis[j];
    const double v2 = __dmul_rn(v, v);
    const int64_t row = ((int64_t)b * side + j) * np;
    for (int k = threadIdx.x; k < np; k += blockDim.x) {
        float2 px = make_float2(0.f, 0.f), py = make_float2(0.f, 0.f);
        if (k < n) {
            const double sx = x[(int64_t)b * n + k];
            const double sy = y[(int64_t)b * n + k];
            const double lens = __dmul_rn(__dmul_rn(c2, z[(int64_t)b * n + k]), v2);
            const double tx = __dadd_rn(__dmul_rn(__dmul_rn(c1, sx), v), lens);
            const double ty = __dadd_rn(__dmul_rn(__dmul_rn(c1, sy), v), lens);
            double s, c;
            sincos(tx, &s, &c);
            px = make_float2((float)c, (float)s);
            sincos(ty, &s, &c);
            py = make_float2((float)c, (float)s);
        }
        gx[row + k] = px;
        gy[row + k] = py;
    }
}

// ---------------------------------------------------------------------------
// Fused pixel pass.  G lanes cooperate on one pixel; lane g owns spots
// n = g + G*k (k < L), so a group's table reads are contiguous.  Each CTA
// owns chunk blockIdx.x of the list ([chunk_len] consecutive entries) for
// pattern blockIdx.y and writes one partial per spot: the per-lane fp32 sums
// are folded over the CTA's pixel slots in slot order.
// ---------------------------------------------------------------------------
template <int G, int L, int MODE>
__global__ void __launch_bounds__(kThreads, (L > 16 ? 1 : 2))
hs_pass_kernel(const PassArgs a)
{
    constexpr int NSLOTS = kThreads / G;
    constexpr bool BWD = (MODE & PM_BWD) != 0;
    constexpr bool FWD = (MODE & PM_FWD) != 0;
    constexpr bool WRITE = (MODE & PM_WRITE) != 0;
    extern __shared__ float2 red[];  // [NSLOTS][np]

    const int pat = blockIdx.y;
    if (a.status != nullptr && a.status[pat] != 0) return;  // uniform per CTA

    const int tid = threadIdx.x;
    const int g = tid % G;
    const int slot = tid / G;
    const int np = a.np;
    const int nl = np / G;
    const float2 *__restrict__ gxp = a.gx + (int64_t)pat * a.tab_stride + g;
    const float2 *__restrict__ gyp = a.gy + (int64_t)pat * a.tab_stride + g;

    float cr[L], ci[L], er[L], ei[L];
#pragma unroll
    for (int k = 0; k < L; ++k) {
        cr[k] = 0.f; ci[k] = 0.f; er[k] = 0.f; ei[k] = 0.f;
        if (BWD && k < nl) {
            const float2 c = a.coef[(int64_t)pat * np + g + G * k];
            cr[k] = c.x; ci[k] = c.y;
        }
    }

    const int64_t begin = (int64_t)blockIdx.x * a.chunk_len;
    int64_t end = begin + a.chunk_len;
    if (end > a.count) end = a.count;
    const int trips = (int)((end - begin + NSLOTS - 1) / NSLOTS);

    for (int t = 0; t < trips; ++t) {
        const int64_t i = begin + (int64_t)t * NSLOTS + slot;
        const bool valid = i < end;
        int rc = 0;
        float A = 0.f;
        if (valid) { rc = __ldg(a.rc + i); A = __ldg(a.amp + i); }
        const int r = rc >> 16, c = rc & 0xffff;
        const float2 *__restrict__ px = gxp + (int64_t)c * np;
        const float2 *__restrict__ py = gyp + (int64_t)r * np;

        float pr[L], pi[L];
        float sr = 0.f, si = 0.f;
#pragma unroll
        for (int k = 0; k < L; ++k) {
            pr[k] = 0.f; pi[k] = 0.f;
            if (k < nl) {
                const float2 u = __ldg(px + G * k);
                const float2 v = __ldg(py + G * k);
                pr[k] = u.x * v.x - u.y * v.y;
                pi[k] = u.x * v.y + u.y * v.x;
                if (BWD) {
                    sr += cr[k] * pr[k] - ci[k] * pi[k];
                    si += cr[k] * pi[k] + ci[k] * pr[k];
                }
            }
        }

        float br, bi;
        if (BWD) {
            // Butterfly over the G lanes of the pixel; a+b == b+a, so every
            // lane ends with the same bits.
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                sr += __shfl_xor_sync(0xffffffffu, sr, o);
                si += __shfl_xor_sync(0xffffffffu, si, o);
            }
            // b = A e^{-i arg S} = A conj(S)/|S|; arg(0) = 0 (kernels.py:115-119).
            const float m2 = sr * sr + si * si;
            if (m2 > 0.f && m2 < INFINITY) {
                const float inv = rsqrtf(m2);
                br = A * (sr * inv);
                bi = -A * (si * inv);
            } else if (sr != 0.f || si != 0.f) {
                const float mx = fmaxf(fabsf(sr), fabsf(si));
                const float xr = sr / mx, xi = si / mx;
                const float inv = rsqrtf(xr * xr + xi * xi);
                br = A * (xr * inv);
                bi = -A * (xi * inv);
            } else {
                br = A;
                bi = 0.f;
            }
            if (WRITE && valid && g == 0) {
                double ph = 0.0;
                if (sr != 0.f || si != 0.f) {
                    ph = (double)atan2f(si, sr);
                    if (ph >= kPi) ph -= kTwoPi;        // pi -> -pi convention
                    else if (ph < -kPi) ph += kTwoPi;   // fp32 -pi below fp64 -pi
                }
                const int64_t di = a.dst ? (int64_t)a.dst[i] : i + a.idx_base;
                a.phase_out[(int64_t)pat * a.phase_stride + di] = ph;
            }
        } else {
            double s = 0.0, co = 1.0;
            if (valid) {
                const int64_t di = a.dst ? (int64_t)a.dst[i] : i + a.idx_base;
                sincos(a.phase_in[(int64_t)pat * a.phase_stride + di], &s, &co);
            }
            br = A * (float)co;
            bi = -A * (float)s;
        }

        if (FWD) {
#pragma unroll
            for (int k = 0; k < L; ++k) {
                er[k] += br * pr[k] - bi * pi[k];
                ei[k] += br * pi[k] + bi * pr[k];
            }
        }
    }

    if (FWD) {
#pragma unroll
        for (int k = 0; k < L; ++k)
            if (k < nl) red[slot * np + g + G * k] = make_float2(er[k], ei[k]);
        __syncthreads();
        float2 *out = a.partials + (int64_t)pat * a.part_stride + (int64_t)blockIdx.x * np;
        for (int n = tid; n < np; n += kThreads) {
            float sx = 0.f, sy = 0.f;
            for (int s = 0; s < NSLOTS; ++s) {
                const float2 v = red[s * np + n];
                sx += v.x;
                sy += v.y;
            }
            out[n] = make_float2(sx, sy);
        }
    }
}

// ---------------------------------------------------------------------------
// Update / epilogue kernel: one CTA per pattern.
// ---------------------------------------------------------------------------
enum UpdMode : int { UPD_SEED = 0, UPD_STEP = 1, UPD_FINAL = 2, UPD_FIELDS = 3 };

struct UpdArgs {
    int mode;
    int n, np, nchunks;
    const float2 *partials;
    int64_t part_stride;
    const double *amp_in;     // [B][n] SEED: amplitudes
    const double *theta_in;   // [B][n] SEED: phase offsets
    const double *a0;         // [B][n] target amplitudes
    double *w;                // [B][np] weights
    float2 *coef;             // [B][np]
    double *trace_w, *trace_m;  // [B][iters][n]
    int iter, iters;
    int32_t *status, *degen, *qstatus;  // [B]
    double *fields;           // [B][n][2]
    double inv_norm;          // 1 / sum_amplitude^2
    double *e, *u, *inten, *rel;  // [B], [B], [B][n], [B][n]
};

__device__ __forceinline__ double hs_wrap(double t)
{
    // optics.py:31-45: exact fmod then one exact +-2pi correction.
    double w = fmod(t, kTwoPi);
    if (w >= kPi) w -= kTwoPi;
    if (w < -kPi) w += kTwoPi;
    return w;
}

// Fixed-shape tree reductions over kUpdThreads values in shared memory.
template <typename T, typename Op>
__device__ __forceinline__ T hs_block_tree(T *buf, T v, Op op)
{
    const int tid = threadIdx.x;
    buf[tid] = v;
    __syncthreads();
    for (int s = kUpdThreads / 2; s > 0; s >>= 1) {
        if (tid < s) buf[tid] = op(buf[tid], buf[tid + s]);
        __syncthreads();
    }
    const T r = buf[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kUpdThreads) hs_update_kernel(const UpdArgs a)
{
    __shared__ double2 fold[kUpdThreads];
    __shared__ double dbuf[kUpdThreads];
    __shared__ int ibuf[kUpdThreads];
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int n = a.n, np = a.np;
    if (a.status[b] != 0) return;

    if (a.mode == UPD_SEED) {
        for (int k = tid; k < np; k += kUpdThreads) {
            float2 c = make_float2(0.f, 0.f);
            double w = 0.0;
            if (k < n) {
                const double th = hs_wrap(a.theta_in[(int64_t)b * n + k]);
                const double am = a.amp_in[(int64_t)b * n + k];
                double s, co;
                sincos(th, &s, &co);
                c = make_float2((float)(am * co), (float)(am * s));
                w = 1.0;
            }
            a.coef[(int64_t)b * np + k] = c;
            if (a.w) a.w[(int64_t)b * np + k] = w;
        }
        return;
    }

    // 1) fold the chunk partials: R ranges per spot, each summed in chunk
    //    order in fp64, then the R range sums in range order.
    int R = kUpdThreads / np;
    if (R < 1) R = 1;
    if (R > a.nchunks) R = a.nchunks;
    const int cpr = (a.nchunks + R - 1) / R;
    const float2 *part = a.partials + (int64_t)b * a.part_stride;
    for (int t = tid; t < R * np; t += kUpdThreads) {
        const int r = t / np, k = t % np;
        const int c0 = r * cpr;
        int c1 = c0 + cpr;
        if (c1 > a.nchunks) c1 = a.nchunks;
        double sx = 0.0, sy = 0.0;
        int c = c0;
        for (; c + 4 <= c1; c += 4) {
            const float2 v0 = part[(int64_t)(c + 0) * np + k];
            const float2 v1 = part[(int64_t)(c + 1) * np + k];
            const float2 v2 = part[(int64_t)(c + 2) * np + k];
            const float2 v3 = part[(int64_t)(c + 3) * np + k];
            sx += (double)v0.x; sy += (double)v0.y;
            sx += (double)v1.x; sy += (double)v1.y;
            sx += (double)v2.x; sy += (double)v2.y;
            sx += (double)v3.x; sy += (double)v3.y;
        }
        for (; c < c1; ++c) {
            const float2 v = part[(int64_t)c * np + k];
            sx += (double)v.x; sy += (double)v.y;
        }
        fold[t] = make_double2(sx, sy);
    }
    __syncthreads();
    double er = 0.0, ei = 0.0;
    const bool live = tid < n;
    if (live) {
        for (int r = 0; r < R; ++r) {
            er += fold[r * np + tid].x;
            ei += fold[r * np + tid].y;
        }
    }
    __syncthreads();

    if (a.mode == UPD_FIELDS || a.mode == UPD_FINAL) {
        if (live) {
            a.fields[((int64_t)b * n + tid) * 2 + 0] = er;
            a.fields[((int64_t)b * n + tid) * 2 + 1] = ei;
        }
        if (a.mode == UPD_FIELDS) return;
        // metrics.py:33-62
        const double I = live ? (er * er + ei * ei) * a.inv_norm : 0.0;
        const double t0 = live ? a.a0[(int64_t)b * n + tid] : 1.0;
        const double rl = I / (t0 * t0);
        if (live) {
            a.inten[(int64_t)b * n + tid] = I;
            a.rel[(int64_t)b * n + tid] = rl;
        }
        const double esum = hs_block_tree(dbuf, I, [](double p, double q) { return p + q; });
        const double hi = hs_block_tree(dbuf, live ? rl : -INFINITY,
                                        [](double p, double q) { return fmax(p, q); });
        const double lo = hs_block_tree(dbuf, live ? rl : INFINITY,
                                        [](double p, double q) { return fmin(p, q); });
        if (tid == 0) {
            a.e[b] = esum;
            if (hi == 0.0) {
                a.u[b] = 0.0;
                a.qstatus[b] = 7;  // HS_EUNDEFINED
            } else {
                a.u[b] = 1.0 - (hi - lo) / (hi + lo);
                a.qstatus[b] = 0;
            }
        }
        return;
    }

    // 2) UPD_STEP: rebalance_weights (solvers.py:104-129) + coefficient
    //    update (solvers.py:148-151, kernels.py:206-208).
    double mag = live ? hypot(er, ei) : 0.0;
    const int zeros = hs_block_tree(ibuf, (live && mag == 0.0) ? 1 : 0,
                                    [](int p, int q) { return p + q; });
    if (zeros > 0) {
        const double minpos = hs_block_tree(dbuf, (live && mag > 0.0) ? mag : INFINITY,
                                            [](double p, double q) { return fmin(p, q); });
        if (minpos == INFINITY) {
            if (tid == 0) a.status[b] = 3;  // HS_EDEGENERATE
            return;
        }
        if (live && mag == 0.0) mag = minpos * 1e-6;  // DEGENERACY_FLOOR
        if (tid == 0 && a.degen[b] == 0) a.degen[b] = a.iter + 1;  // first degenerate step
    }
    const double msum = hs_block_tree(dbuf, live ? mag : 0.0,
                                      [](double p, double q) { return p + q; });
    const double mean = msum / (double)n;
    double w = 0.0;
    if (live) w = a.w[(int64_t)b * np + tid] * (mean / mag);
    const int bad = hs_block_tree(ibuf, (live && !isfinite(w)) ? 1 : 0,
                                  [](int p, int q) { return p + q; });
    if (bad > 0) {
        if (tid == 0) a.status[b] = 4;  // HS_EDIVERGED
        return;
    }
    if (live) {
        const int64_t tix = ((int64_t)b * a.iters + a.iter) * n + tid;
        a.trace_w[tix] = w;
        a.trace_m[tix] = mag;
        a.w[(int64_t)b * np + tid] = w;
        const double am = w * a.a0[(int64_t)b * n + tid];
        double th = 0.0;
        if (er != 0.0 || ei != 0.0) {
            th = atan2(ei, er);
            if (th == kPi) th = -kPi;
        }
        double s, co;
        sincos(th, &s, &co);
        a.coef[(int64_t)b * np + tid] = make_float2((float)(am * co), (float)(am * s));
    }
}

}  // namespace hs
