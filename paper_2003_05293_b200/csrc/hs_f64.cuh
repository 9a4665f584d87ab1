// hs_f64.cuh -- the fp64 pixel passes (precision "fp64").
//
// Same schedule, fold and update as the fp32 passes, but every pixel-spot
// product, the per-pixel field S_p, the illumination amplitude, the tables
// and the coefficients are fp64, as in the reference kernels
// (holospots/kernels.py:78-144, fp64 numba):
//
//   hs_tables64_kernel  gx, gy as fp64 unit phasors (kernels.py:78-96; no
//                       rounding to fp32), seed coefficients in fp64
//   hs_pass64_kernel    one CTA per chunk of a storage-order pixel range:
//                       phase A (one warp per pixel, lanes over spots)
//                         S_p = sum_n (coef_n gx[c_p,n]) gy[r_p,n]
//                         -> b_p = A_p conj(S_p)/|S_p|, arg S_p on the final
//                            pass (kernels.py:99-119);
//                         or b_p = A_p e^{-i phi_p} from a given phase
//                            (forward only, kernels.py:135-139);
//                       phase B (one thread per spot, pixels in storage order)
//                         E_n += b_p (gx[c_p,n] gy[r_p,n]) (kernels.py:140-144)
//                       then the fixed two-level fold and the update
//                       (hs_fold with fp64 partials).
//
// Why it exists: WGS amplifies per-iteration rounding noise by a factor that
// grows as the problem gets less overdetermined (few pixels per spot in a
// window).  At >= 512 pixels per spot the fp32 passes stay >10x inside the
// north-star tolerances (config 3: 651, config 4: 1042); below that the fp32
// accumulation noise (~1e-6 relative at iteration 1) grows ~3-5x per
// iteration and reaches 1e-4 within a few iterations on e.g. 600 spots on a
// 256^2 pupil (tools/accuracy_probe.py).  The solver
// picks these kernels automatically there (precision "auto"); they also
// carry spot counts above the fp32 kernels' 1024.
//
// Determinism: the per-pixel sum is a fixed butterfly (commutative pairs, all
// lanes identical bits), the per-chunk sum runs in storage order, the fold is
// the fixed two-level tree -- bitwise run-to-run and batch-invariant.
#pragma once

#include "hs_kernels.cuh"

namespace hs {

constexpr int kP64Threads = 256;
constexpr int kP64Warps = kP64Threads / 32;
constexpr int kP64SpotsPerThread = 4;   // phase B register accumulators per spot sweep

struct Pass64Args {
    const int32_t *rc;        // storage list (row << 16) | col
    const double *amp;        // storage-order illumination amplitude (fp64)
    int64_t start;            // first storage pixel of the range
    int64_t count;            // pixels in the range
    int32_t chunk_len;        // pixels per CTA
    int32_t n, np;            // spots, table row stride
    int64_t tab_stride;       // side * np
    const double2 *gx, *gy;   // [B][side][np]
    const double2 *coef;      // [B][np]
    const double *phase_in;   // [B][phase_stride] (forward-only passes)
    double *phase_out;        // [B][phase_stride] (PM_WRITE)
    unsigned char *raster;    // [B][side][side] SLM gray raster (PM_WRITE, nullable)
    int32_t side;
    int64_t phase_stride;
    FoldArgs f;               // f.partials64
};

__host__ __device__ constexpr size_t hs_pass64_smem_bytes(int np, int chunk_len)
{
    // coef [np] + b [chunk] (double2) + rc [chunk]; the fold's scratch needs
    // np double2 + 2 np double
    return (16 * (size_t)np + 20 * (size_t)chunk_len) > 32 * (size_t)np
               ? 16 * (size_t)np + 20 * (size_t)chunk_len
               : 32 * (size_t)np;
}

static __global__ void hs_tables64_kernel(int side, int np, int n, const double *__restrict__ axis, double c1,
                                          double c2, const double *__restrict__ x, const double *__restrict__ y,
                                          const double *__restrict__ z, double2 *__restrict__ gx,
                                          double2 *__restrict__ gy, const double *seed_amp,
                                          const double *seed_theta, double2 *coef, double *w)
{
    const int j = blockIdx.x;
    const int b = blockIdx.y;
    const double v = axis[j];
    const double v2 = __dmul_rn(v, v);
    const int64_t row = ((int64_t)b * side + j) * np;
    for (int k = threadIdx.x; k < np; k += blockDim.x) {
        double2 px = make_double2(0.0, 0.0), py = make_double2(0.0, 0.0);
        if (k < n) {
            // kernels.py:88-94, the reference's operation order
            const double sx = x[(int64_t)b * n + k];
            const double sy = y[(int64_t)b * n + k];
            const double lens = __dmul_rn(__dmul_rn(c2, z[(int64_t)b * n + k]), v2);
            const double tx = __dadd_rn(__dmul_rn(__dmul_rn(c1, sx), v), lens);
            const double ty = __dadd_rn(__dmul_rn(__dmul_rn(c1, sy), v), lens);
            sincos(tx, &px.y, &px.x);
            sincos(ty, &py.y, &py.x);
        }
        gx[row + k] = px;
        gy[row + k] = py;
        if (j == 0 && seed_theta != nullptr) hs_seed_one(b, k, n, np, seed_amp, seed_theta, nullptr, w, coef);
    }
}

template <int MODE>
__global__ void __launch_bounds__(kP64Threads) hs_pass64_kernel(const Pass64Args a)
{
    constexpr bool BWD = (MODE & PM_BWD) != 0;
    constexpr bool FWD = (MODE & PM_FWD) != 0;
    constexpr bool WRITE = (MODE & PM_WRITE) != 0;
    extern __shared__ double2 sm64[];
    const int pat = blockIdx.y;
    const int chunk = a.f.chunk_base + blockIdx.x;
    hs_pdl_wait_prev();    // previous pass's fold / update visible (no-op for a plain launch)
    hs_pdl_launch_next();
    if (a.f.u.status[pat] != 0) return;  // pattern already failed (uniform per CTA)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int np = a.np, L = a.chunk_len;
    double2 *coef_s = sm64;                                        // [np]
    double2 *b_s = sm64 + np;                                      // [L]
    int32_t *rc_s = reinterpret_cast<int32_t *>(b_s + L);          // [L]
    const int64_t p0 = a.start + (int64_t)chunk * L;
    const int64_t rem = a.start + a.count - p0;
    const int len = rem < (int64_t)L ? (int)rem : L;

    for (int i = tid; i < len; i += kP64Threads) rc_s[i] = __ldg(a.rc + p0 + i);
    if (BWD)
        for (int k = tid; k < np; k += kP64Threads) coef_s[k] = a.coef[(int64_t)pat * np + k];
    __syncthreads();

    const double2 *__restrict__ gx = a.gx + (int64_t)pat * a.tab_stride;
    const double2 *__restrict__ gy = a.gy + (int64_t)pat * a.tab_stride;

    // phase A: per pixel b_p (one warp per pixel)
    for (int i = warp; i < len; i += kP64Warps) {
        const int rc = rc_s[i], r = rc >> 16, c = rc & 0xffff;
        const double A = __ldg(a.amp + p0 + i);
        double2 b;
        if (BWD) {
            const double2 *xr = gx + (int64_t)c * np, *yr = gy + (int64_t)r * np;
            double sr = 0.0, si = 0.0;
            for (int k = lane; k < a.n; k += 32) {
                const double2 q = __ldg(xr + k), v = __ldg(yr + k), cf = coef_s[k];
                // u = gx * coef (kernels.py:206-210), S += u * gy (kernels.py:108-113)
                const double ur = q.x * cf.x - q.y * cf.y;
                const double ui = q.x * cf.y + q.y * cf.x;
                sr += ur * v.x - ui * v.y;
                si += ur * v.y + ui * v.x;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sr += __shfl_xor_sync(0xffffffffu, sr, o);
                si += __shfl_xor_sync(0xffffffffu, si, o);
            }
            if (sr == 0.0 && si == 0.0) {
                b = make_double2(A, 0.0);                          // arg(0) = 0 (kernels.py:115-116)
            } else {
                const double m = hypot(sr, si);
                b = make_double2(A * (sr / m), -A * (si / m));     // A e^{-i arg S}
            }
            if (WRITE && lane == 0) {
                double ph = 0.0;
                if (sr != 0.0 || si != 0.0) {
                    ph = atan2(si, sr);                            // kernels.py:117-119
                    if (ph == kPi) ph = -kPi;
                }
                a.phase_out[(int64_t)pat * a.phase_stride + p0 + i] = ph;
                if (a.raster) a.raster[(int64_t)pat * a.side * a.side + (int64_t)r * a.side + c] = hs_gray_linear(ph);
            }
        } else {
            double sn, cs;
            sincos(a.phase_in[(int64_t)pat * a.phase_stride + p0 + i], &sn, &cs);
            b = make_double2(A * cs, -A * sn);                     // kernels.py:137-139
        }
        if (lane == 0) b_s[i] = b;
    }
    if (!FWD) return;
    __syncthreads();

    // phase B: per spot, pixels in storage order (kernels.py:140-144)
    double2 *out = a.f.partials64 + (int64_t)pat * a.f.part_stride + (int64_t)chunk * np;
    constexpr int SPT = kP64SpotsPerThread;
    for (int k0 = 0; k0 < np; k0 += kP64Threads * SPT) {
        double er[SPT], ei[SPT];
#pragma unroll
        for (int j = 0; j < SPT; ++j) { er[j] = 0.0; ei[j] = 0.0; }
        for (int i = 0; i < len; ++i) {
            const int rc = rc_s[i];
            const double2 b = b_s[i];
            const double2 *xr = gx + (int64_t)(rc & 0xffff) * np, *yr = gy + (int64_t)(rc >> 16) * np;
#pragma unroll
            for (int j = 0; j < SPT; ++j) {
                const int k = k0 + tid + j * kP64Threads;
                if (k < a.n) {
                    const double2 q = __ldg(xr + k), v = __ldg(yr + k);
                    const double tr = q.x * v.x - q.y * v.y;
                    const double ti = q.x * v.y + q.y * v.x;
                    er[j] += b.x * tr - b.y * ti;
                    ei[j] += b.x * ti + b.y * tr;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            const int k = k0 + tid + j * kP64Threads;
            if (k < np) out[k] = make_double2(er[j], ei[j]);
        }
    }
    if (a.f.u.act != ACT_NONE) {
        __syncthreads();
        hs_fold(a.f, pat, chunk, reinterpret_cast<char *>(sm64));
    }
}

// user tables (hs_set_tables / hs_get_tables): [side][n] re/im planes <-> [side][np] phasors
static __global__ void hs_pack_tables_kernel(int side, int n, int np, const double *re, const double *im,
                                             double2 *t64, float2 *t32)
{
    const int j = blockIdx.x;
    for (int k = threadIdx.x; k < np; k += blockDim.x) {
        const double2 v = k < n ? make_double2(re[(int64_t)j * n + k], im[(int64_t)j * n + k])
                                : make_double2(0.0, 0.0);
        t64[(int64_t)j * np + k] = v;
        t32[(int64_t)j * np + k] = make_float2((float)v.x, (float)v.y);
    }
}

static __global__ void hs_unpack_tables_kernel(int side, int n, int np, const double2 *t64, double *re,
                                               double *im)
{
    const int j = blockIdx.x;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const double2 v = t64[(int64_t)j * np + k];
        re[(int64_t)j * n + k] = v.x;
        im[(int64_t)j * n + k] = v.y;
    }
}

typedef void (*Pass64Fn)(Pass64Args);

inline Pass64Fn hs_select_pass64(int mode)
{
    switch (mode) {
    case PM_BWD | PM_WRITE: return hs_pass64_kernel<PM_BWD | PM_WRITE>;
    case PM_FWD: return hs_pass64_kernel<PM_FWD>;
    case PM_BWD | PM_FWD: return hs_pass64_kernel<PM_BWD | PM_FWD>;
    case PM_BWD | PM_FWD | PM_WRITE: return hs_pass64_kernel<PM_BWD | PM_FWD | PM_WRITE>;
    default: return nullptr;
    }
}

}  // namespace hs
