// hs_kernels.cuh -- sm_100a device kernels of the CS-WGS hot path.
//
//   hs_tables_kernel  per-pattern column/row unit phasors gx, gy
//                     (reference _build_tables, holospots/kernels.py:78-96),
//                     optionally fused with the seed coefficients
//                     (solvers.py:166-176, kernels.py:206-208)
//   hs_seed_kernel    superposition coefficients a e^{i wrap(theta)}
//   hs_pass_kernel    fused pixel pass over a pixel list:
//                       back-propagation S_p = sum_n coef_n gy[r_p,n] gx[c_p,n]
//                       -> arg S_p (kernels.py:99-119), and/or
//                       forward projection E_n += b_p gx[c_p,n] gy[r_p,n] with
//                       b_p = A_p e^{-i arg S_p} (kernels.py:122-144);
//                     then a two-level fixed-order fold of the per-CTA partials
//                     done by the last CTA of each group / pattern, which also
//                     runs the weight / theta update (solvers.py:104-163) or the
//                     e / u epilogue (metrics.py:33-79) -- one launch per
//                     solver iteration.
//
// Work decomposition.  G lanes cooperate on one pixel;
// lane g owns spots {2g, 2g+1} + 2G*j (j < nl/2) so table rows are read as
// float4.  A warp holds SPW = 32/G pixel slots.  Each slot walks a run of
// list entries; while the row stays the same it keeps V = coef * gy[row]
// (backward) and T = sum b_p gx[c_p] (forward) in registers, so a pixel
// costs one gx row read + 8 FFMA per spot, and a row change costs one gy
// row read.  Dense (full-range) lists are laid out so the SPW slots of a warp
// sit on SPW rows of the same column(s): the gx row load is a broadcast.
//
// Numerics: phasor arguments are formed in fp64 in the reference's order
// (no FMA contraction) and rounded to fp32 phasors; pixel loops run in fp32
// on the FMA pipe; every cross-pixel reduction has a fixed shape that
// depends only on the list layout, so results are bitwise reproducible and
// independent of the batch size and of CTA scheduling.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hs {

constexpr int kThreads = 256;        // pass-kernel CTA size (8 warps)
constexpr int kWarps = kThreads / 32;
constexpr int kTargetChunks = 296;   // sparse lists: chunks per pattern (2 x 148 SMs)
// Timing probes inside the pass kernels (HS_SLAB_TRACE / HS_UMMA_TRACE with
// hs_time_kernel) are compiled in only with -DHS_PROBES=1 (build.py: HS_PROBES=1
// in the environment); compiled out they cost nothing (2-3% of the tcgen05
// pass when present).
#ifndef HS_PROBES
#define HS_PROBES 0
#endif

constexpr int kGroup = 32;           // chunks per first-level fold group
constexpr int kFoldBatch = 16;       // partial loads in flight per thread in the group fold
constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 6.283185307179586;

enum PassMode : int { PM_BWD = 1, PM_FWD = 2, PM_WRITE = 4 };
enum FoldAct : int { ACT_NONE = 0, ACT_STEP = 1, ACT_FINAL = 2, ACT_FIELDS = 3 };

struct UpdArgs {
    int act;                  // FoldAct
    int n, np;
    const double *a0;         // [B][n] target amplitudes
    double *w;                // [B][np] weights
    float2 *coef;             // [B][np] coefficients for the next pass (fp32 passes)
    double2 *coef64;          // [B][np] the same in fp64 (fp64 passes; coef unused)
    double *trace_w, *trace_m;  // [B][iters][n]
    int iter, iters;
    int32_t *status, *degen, *qstatus;  // [B]
    double *fields;           // [B][n][2]
    double inv_norm;          // 1 / sum_amplitude^2
    double *e, *u, *inten, *rel;  // [B], [B], [B][n], [B][n]
};

// Cross-CTA fold state shared by the pass and tile kernels.
struct FoldArgs {
    int32_t nchunks;          // partials per pattern in this launch
    int32_t chunk_base;       // first chunk of this launch (row-sharded passes)
    int32_t chunk_end;        // one past the last chunk of this launch
    int32_t np;
    float2 *partials;         // [B][part_stride]: [chunk][np] (fp32 passes)
    double2 *partials64;      // the same layout in fp64 (fp64 passes; partials unused)
    int64_t part_stride;
    double2 *gpart;           // [B][gpart_stride]: [group][np]
    int64_t gpart_stride;
    int32_t *grp_cnt;         // [B][cnt_stride] arrival counters (self-resetting)
    int32_t *pat_cnt;         // [B]
    int32_t cnt_stride;
    UpdArgs u;
};

struct PassArgs {
    const int32_t *rc;        // packed (row << 16) | col per list entry
    const float *amp;         // illumination amplitude per entry (0: padding)
    const int32_t *dst;       // storage index per entry, -1 padding (nullptr: i + idx_base)
    int64_t idx_base;
    int64_t count;            // list length
    int32_t chunk_len;        // entries per CTA; multiple of 8 * SPW
    int32_t np, nl;           // padded spot count, spots per lane (even)
    int32_t sorted_rows;      // list is sorted by row (window lists)
    int64_t tab_stride;       // side * np
    const float2 *gx, *gy;    // [B][side][np]
    const float2 *coef;       // [B][np]
    const double *phase_in;   // [B][phase_stride] (PM_FWD without PM_BWD)
    double *phase_out;        // [B][phase_stride] (PM_WRITE)
    float *phase_out32;       // the same as 4-byte phase codes (PM_WRITE; replaces phase_out)
    unsigned char *raster;    // [B][side][side] SLM gray raster (PM_WRITE, nullable)
    int32_t side;
    int64_t phase_stride;
    FoldArgs f;
};

// ---------------------------------------------------------------------------
// Programmatic dependent launch (the pass kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization inside the solve graph):
// a pass lets the next pass launch as soon as all its CTAs are resident, and
// the next pass stages its static inputs (gx slab, pixel lists) before
// waiting for the previous pass's fold / update to complete and become
// visible.  Both are no-ops for a normal launch.
__device__ __forceinline__ void hs_pdl_launch_next()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint32_t hs_smem_addr(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void hs_pdl_wait_prev()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ double hs_wrap(double t)
{
    // optics.py:31-45: exact fmod, then one exact +-2pi correction.
    double w = fmod(t, kTwoPi);
    if (w >= kPi) w -= kTwoPi;
    if (w < -kPi) w += kTwoPi;
    return w;
}

// Stored phase of a pixel: arg S from fp32 atan2f, widened to f64 and wrapped
// to [-pi, pi) with pi -> -pi (optics.py:31-45, solvers.py:96-101), arg(0) =
// 0.  atan2f's range is [-pi_f32, pi_f32] and pi_f32 > pi_f64, so the only
// widened values outside [-pi, pi) are +-pi_f32 themselves: the wrap is
// decided in fp32 and its two results are the fp64 constants pi_f32 - 2 pi
// and -pi_f32 + 2 pi (the same bits as wrapping the widened value).
// atan2 for finite (y, x) != (0, 0): octant reduction r = min/max in [0, 1],
// atan(r) = r P(r^2) with a degree-8 least-squares fit (max |error| of the
// fp32 evaluation 2.8e-7 rad over 2M random points, the same as fp32 atan2's
// own; fitted by tools/atan2_fit.py), then the quadrant fix-ups.  About half
// the instructions of atan2f (no IEEE division).  Signed zeros as atan2:
// atan2(+0, x < 0) = +pi_f32, atan2(-0, x < 0) = -pi_f32.
__device__ __forceinline__ float hs_atan2(float y, float x)
{
    const float ax = fabsf(x), ay = fabsf(y);
    float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    if (mx < 1.0e-30f) {  // keep 1 / mx finite for tiny (denormal) arguments
        mx *= 18446744073709551616.0f;
        mn *= 18446744073709551616.0f;
    }
    const float r = mn * __frcp_rn(mx);
    const float s = r * r;
    float p = 0.0029035801999270916f;
    p = fmaf(p, s, -0.016283102333545685f);
    p = fmaf(p, s, 0.04303948953747749f);
    p = fmaf(p, s, -0.07533683627843857f);
    p = fmaf(p, s, 0.1065467968583107f);
    p = fmaf(p, s, -0.14207133650779724f);
    p = fmaf(p, s, 0.19993053376674652f);
    p = fmaf(p, s, -0.3333309292793274f);
    p = fmaf(p, s, 1.0f);
    float a = r * p;
    if (ay > ax) a = 1.57079637050628662f - a;
    if (x < 0.f) a = 3.14159274101257324f - a;
    return copysignf(a, y);
}

__device__ __forceinline__ double hs_phase_f64(float x, float y)
{
    if (x == 0.f && y == 0.f) return 0.0;
    const float p = hs_atan2(y, x);
    if (p == 3.14159274101257324f) return 3.14159274101257324 - kTwoPi;
    if (p == -3.14159274101257324f) return -3.14159274101257324 + kTwoPi;
    return (double)p;
}

// The 4-byte phase code the f64 phase is a fixed function of: the fp32 atan2
// (0 for S = 0).  hs_widen_phase (host, hs_plan.cu) maps it back to exactly
// hs_phase_f64's value, so solves can ship half the bytes to the host.
__device__ __forceinline__ float hs_phase_code(float x, float y)
{
    return (x == 0.f && y == 0.f) ? 0.f : hs_atan2(y, x);
}

// hs_phase_f64's value from its code (the host twin is hs_widen_phases).
__host__ __device__ __forceinline__ double hs_widen_code(float p)
{
    if (p == 3.14159274101257324f) return 3.14159274101257324 - kTwoPi;
    if (p == -3.14159274101257324f) return -3.14159274101257324 + kTwoPi;
    return (double)p;
}

static __global__ void hs_widen_codes_kernel(const float *__restrict__ src, double *__restrict__ dst, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = hs_widen_code(src[i]);
}

// Store one pixel's phase: the f64 value, or its 4-byte code when the pass
// writes codes (phase_out32 != nullptr).
__device__ __forceinline__ void hs_store_phase(double *out, float *out32, int64_t idx, float x, float y)
{
    if (out32) out32[idx] = hs_phase_code(x, y);
    else out[idx] = hs_phase_f64(x, y);
}

// Linear phase -> gray lookup of the default PhaseLut (fileio.py:159-213):
// g = rint((p + pi) * 256 / (2 pi)) mod 256 on the wrapped fp64 phase, with
// the reference's operation order (no contraction), so a device raster equals
// PhaseLut.default().gray(phase) bit for bit.
__device__ __forceinline__ unsigned char hs_gray_linear(double p)
{
    const double g = rint(__dmul_rn(__dadd_rn(p, kPi), 256.0 / kTwoPi));
    return (unsigned char)(((long long)g) & 255);
}

// coef = a e^{i wrap(theta)} (kernels.py:206-208); fp32 (coef) or fp64 (coef64)
__device__ __forceinline__ void hs_seed_one(int b, int k, int n, int np, const double *amp,
                                            const double *theta, float2 *coef, double *w,
                                            double2 *coef64 = nullptr)
{
    double2 c = make_double2(0.0, 0.0);
    double wk = 0.0;
    if (k < n) {
        const double th = hs_wrap(theta[(int64_t)b * n + k]);
        const double am = amp[(int64_t)b * n + k];
        double s, co;
        sincos(th, &s, &co);
        c = make_double2(am * co, am * s);
        wk = 1.0;
    }
    if (coef64) coef64[(int64_t)b * np + k] = c;
    else coef[(int64_t)b * np + k] = make_float2((float)c.x, (float)c.y);
    if (w) w[(int64_t)b * np + k] = wk;
}

// Tables: gx[b][j][n] = exp(i (c1 x_n a_j + c2 z_n a_j^2)), gy likewise with
// y_n; the argument is formed with explicit round-to-nearest fp64 ops in the
// reference order ((c1*x)*v + (c2*z)*v2) -> numba's bits; fp64 sincos; one
// rounding to fp32.  Block (0, b) also seeds pattern b when seed_theta != 0.
static __global__ void hs_tables_kernel(int side, int np, int n, const double *__restrict__ axis,
                                 double c1, double c2, const double *__restrict__ x,
                                 const double *__restrict__ y, const double *__restrict__ z,
                                 float2 *__restrict__ gx, float2 *__restrict__ gy,
                                 const double *seed_amp, const double *seed_theta,
                                 float2 *coef, double *w)
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
        if (j == 0 && seed_theta != nullptr) hs_seed_one(b, k, n, np, seed_amp, seed_theta, coef, w);
    }
}

static __global__ void hs_seed_kernel(int n, int np, const double *amp, const double *theta, float2 *coef,
                               double *w, double2 *coef64 = nullptr)
{
    for (int k = threadIdx.x; k < np; k += blockDim.x)
        hs_seed_one(blockIdx.x, k, n, np, amp, theta, coef, w, coef64);
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ float hs_rsqrt(float x)
{
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// b = A conj(S)/|S| with arg(0) = 0 (kernels.py:136-137, solvers.py:96-101)
__device__ __forceinline__ void hs_bvec(float sr, float si, float A, float &br, float &bi)
{
    const float m2 = fmaf(sr, sr, si * si);
    if (__float_as_uint(m2) - 0x0d800000u < 0x64000000u) {  // 2^-100 <= m2 < 2^100
        const float inv = A * hs_rsqrt(m2);
        br = sr * inv;
        bi = -si * inv;
    } else if (sr != 0.f || si != 0.f) {
        const float mx = fmaxf(fabsf(sr), fabsf(si));
        const float xr = sr / mx, xi = si / mx;
        const float inv = A * hs_rsqrt(fmaf(xr, xr, xi * xi));
        br = xr * inv;
        bi = -xi * inv;
    } else {
        br = A;
        bi = 0.f;
    }
}

// hs_bvec without branches: S is scaled by the power of two 2^-e that
// brings max(|Sr|, |Si|) into [1, 2) before |S|^2 is formed.  Scaling by a
// power of two is exact, so wherever hs_bvec takes its fast path the result
// is bitwise the same; tiny and huge |S| need no separate path.
__device__ __forceinline__ void hs_bvec_nb(float sr, float si, float A, float &br, float &bi)
{
    const float mx = fmaxf(fabsf(sr), fabsf(si));
    const float sc = __int_as_float(0x7f000000 - (__float_as_int(mx) & 0x7f800000));  // 2^-e (2^127 for denormals)
    const float xr = sr * sc, xi = si * sc;
    const float inv = A * hs_rsqrt(fmaf(xr, xr, xi * xi));
    br = mx > 0.f ? xr * inv : A;
    bi = mx > 0.f ? -xi * inv : 0.f;
}

// Fixed-shape block reductions over kThreads values: a butterfly inside each
// warp (every lane ends with the same bits: the pairs are commutative), then
// the kWarps warp results combined in warp order.  Deterministic and ~4x
// shallower than a shared-memory tree.
template <typename T, typename Op>
__device__ __forceinline__ T hs_tree(T *buf, T v, Op op)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int tid = threadIdx.x;
    if ((tid & 31) == 0 && tid < kThreads) buf[tid >> 5] = v;
    __syncthreads();
    T r = buf[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) r = op(r, buf[w]);
    __syncthreads();
    return r;
}

struct DSum { __device__ double operator()(double p, double q) const { return p + q; } };
struct DMin { __device__ double operator()(double p, double q) const { return fmin(p, q); } };
struct DMax { __device__ double operator()(double p, double q) const { return fmax(p, q); } };
struct ISum { __device__ int operator()(int p, int q) const { return p + q; } };

// Threads of a CTA that take part in the fold / update arithmetic: the first
// kThreads (wider CTAs only join the barriers), so every kernel folds and
// updates with the same reduction order -- bitwise identical results.
__device__ __forceinline__ int hs_team_tid()
{
    return threadIdx.x < kThreads ? (int)threadIdx.x : (1 << 29);
}

// The pattern's fields E (fp64, in shared memory) -> action.  Runs in the
// last CTA of the pattern (kThreads team; all threads reach the barriers).
__device__ __forceinline__ void hs_update(const UpdArgs &a, int b, double2 *E, double *mag_s,
                                       double *dbuf, int *ibuf)
{
    const int tid = hs_team_tid();
    const int n = a.n, np = a.np;
    if (a.act == ACT_FIELDS || a.act == ACT_FINAL) {
        double esum = 0.0, hi = -INFINITY, lo = INFINITY;
        for (int k = tid; k < n; k += kThreads) {
            const double er = E[k].x, ei = E[k].y;
            a.fields[((int64_t)b * n + k) * 2 + 0] = er;
            a.fields[((int64_t)b * n + k) * 2 + 1] = ei;
            if (a.act == ACT_FINAL) {
                const double I = (er * er + ei * ei) * a.inv_norm;   // metrics.py:33-42
                const double t0 = a.a0[(int64_t)b * n + k];
                const double rl = I / (t0 * t0);                     // metrics.py:65-68
                a.inten[(int64_t)b * n + k] = I;
                a.rel[(int64_t)b * n + k] = rl;
                esum += I;
                hi = fmax(hi, rl);
                lo = fmin(lo, rl);
            }
        }
        if (a.act == ACT_FIELDS) return;
        esum = hs_tree(dbuf, esum, DSum());                          // metrics.py:45-50
        hi = hs_tree(dbuf, hi, DMax());
        lo = hs_tree(dbuf, lo, DMin());
        if (tid == 0) {
            a.e[b] = esum;
            if (hi == 0.0) {                                         // metrics.py:53-62
                a.u[b] = 0.0;
                a.qstatus[b] = 7;  // HS_EUNDEFINED
            } else {
                a.u[b] = 1.0 - (hi - lo) / (hi + lo);
                a.qstatus[b] = 0;
            }
        }
        return;
    }
    // ACT_STEP: rebalance_weights (solvers.py:104-129), then the coefficient
    // update a = w a0, theta = arg E (solvers.py:148-151, kernels.py:206-208).
    // theta and its sincos depend on E alone: they are computed in the first
    // loop (E[k] is replaced by (cos, sin)), off the chain of reductions.
    int zeros = 0;
    double minpos = INFINITY, msum = 0.0;
    for (int k = tid; k < n; k += kThreads) {
        const double er = E[k].x, ei = E[k].y;
        const double m = hypot(er, ei);
        mag_s[k] = m;
        if (m == 0.0) ++zeros;
        else minpos = fmin(minpos, m);
        msum += m;
        double th = 0.0;                                   // solvers.py:96-101
        if (er != 0.0 || ei != 0.0) {
            th = atan2(ei, er);
            if (th == kPi) th = -kPi;
        }
        double sn, co;
        sincos(th, &sn, &co);
        E[k] = make_double2(co, sn);
    }
    zeros = hs_tree(ibuf, zeros, ISum());
    if (zeros > 0) {
        minpos = hs_tree(dbuf, minpos, DMin());
        if (minpos == INFINITY) {
            if (tid == 0) a.status[b] = 3;  // HS_EDEGENERATE
            return;
        }
        msum = 0.0;
        for (int k = tid; k < n; k += kThreads) {
            if (mag_s[k] == 0.0) mag_s[k] = minpos * 1e-6;  // DEGENERACY_FLOOR
            msum += mag_s[k];
        }
        if (tid == 0 && a.degen[b] == 0) a.degen[b] = a.iter + 1;
    }
    msum = hs_tree(dbuf, msum, DSum());
    const double mean = msum / (double)n;
    int bad = 0;
    for (int k = tid; k < n; k += kThreads) {
        const double wk = a.w[(int64_t)b * np + k] * (mean / mag_s[k]);
        if (!isfinite(wk)) ++bad;
        mag_s[k + np] = wk;  // stash (mag_s has 2*np doubles)
    }
    bad = hs_tree(ibuf, bad, ISum());
    if (bad > 0) {
        if (tid == 0) a.status[b] = 4;  // HS_EDIVERGED
        return;
    }
    for (int k = tid; k < n; k += kThreads) {
        const double wk = mag_s[k + np];
        const int64_t tix = ((int64_t)b * a.iters + a.iter) * n + k;
        a.trace_w[tix] = wk;
        a.trace_m[tix] = mag_s[k];
        a.w[(int64_t)b * np + k] = wk;
        const double am = wk * a.a0[(int64_t)b * n + k];
        const double co = E[k].x, sn = E[k].y;
        if (a.coef64) a.coef64[(int64_t)b * np + k] = make_double2(am * co, am * sn);
        else a.coef[(int64_t)b * np + k] = make_float2((float)(am * co), (float)(am * sn));
    }
}

// Two-level fold run after a CTA has written its chunk partial.  The last CTA
// of each kGroup-chunk group folds the group in chunk order (fp64); the last
// group-folder of the pattern folds the groups in order and applies the
// action.  Counters reset themselves, so graphs replay without memsets.
__device__ __forceinline__ void hs_fold(const FoldArgs &a, int pat, int chunk, char *scratch, int arrivals = 1)
{
    __shared__ int s_last;
    __shared__ double dbuf[kThreads];
    __shared__ int ibuf[kThreads];
    const int tid = hs_team_tid();
    const int np = a.np;
    const int ngroups = (a.nchunks + kGroup - 1) / kGroup;
    const int grp = chunk / kGroup;
    const int c0 = grp * kGroup;
    const int c1 = min(c0 + kGroup, a.nchunks);
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const int t = atomicAdd(a.grp_cnt + (int64_t)pat * a.cnt_stride + grp, arrivals);
        s_last = (t + arrivals == c1 - c0);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double2 *gp = a.gpart + (int64_t)pat * a.gpart_stride;
    // Loads are issued kFoldBatch at a time ahead of the (chunk-ordered) sums: a few L2
    // round trips on the fold tail instead of c1 - c0 dependent ones.
    if (a.partials64) {
        const double2 *part = a.partials64 + (int64_t)pat * a.part_stride;
        for (int k = tid; k < np; k += kThreads) {
            double sx = 0.0, sy = 0.0;
            for (int cb = c0; cb < c1; cb += kFoldBatch) {
                double2 v[kFoldBatch];
#pragma unroll
                for (int c = 0; c < kFoldBatch; ++c)
                    if (cb + c < c1) v[c] = __ldcg(part + (int64_t)(cb + c) * np + k);
#pragma unroll
                for (int c = 0; c < kFoldBatch; ++c)
                    if (cb + c < c1) {
                        sx += v[c].x;
                        sy += v[c].y;
                    }
            }
            gp[(int64_t)grp * np + k] = make_double2(sx, sy);
        }
    } else {
        const float2 *part = a.partials + (int64_t)pat * a.part_stride;
        for (int k = tid; k < np; k += kThreads) {
            double sx = 0.0, sy = 0.0;
            for (int cb = c0; cb < c1; cb += kFoldBatch) {
                float2 v[kFoldBatch];
#pragma unroll
                for (int c = 0; c < kFoldBatch; ++c)
                    if (cb + c < c1) v[c] = __ldcg(part + (int64_t)(cb + c) * np + k);
#pragma unroll
                for (int c = 0; c < kFoldBatch; ++c)
                    if (cb + c < c1) {
                        sx += (double)v[c].x;
                        sy += (double)v[c].y;
                    }
            }
            gp[(int64_t)grp * np + k] = make_double2(sx, sy);
        }
    }
    if (tid == 0) a.grp_cnt[(int64_t)pat * a.cnt_stride + grp] = 0;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const int t = atomicAdd(a.pat_cnt + pat, 1);
        s_last = (t == ngroups - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (tid == 0) a.pat_cnt[pat] = 0;
    double2 *E = reinterpret_cast<double2 *>(scratch);           // [np]
    double *mag_s = reinterpret_cast<double *>(E + np);           // [2*np]
    for (int k = tid; k < np; k += kThreads) {
        double sx = 0.0, sy = 0.0;
        for (int g0 = 0; g0 < ngroups; g0 += 8) {  // 8 loads in flight, summed in group order
            double2 v[8];
#pragma unroll
            for (int gI = 0; gI < 8; ++gI)
                if (g0 + gI < ngroups) v[gI] = __ldcg(gp + (int64_t)(g0 + gI) * np + k);
#pragma unroll
            for (int gI = 0; gI < 8; ++gI)
                if (g0 + gI < ngroups) {
                    sx += v[gI].x;
                    sy += v[gI].y;
                }
        }
        E[k] = make_double2(sx, sy);
    }
    __syncthreads();
    hs_update(a.u, pat, E, mag_s, dbuf, ibuf);
}

// ---------------------------------------------------------------------------
constexpr int kMaxChunk = 2048;  // largest chunk_len of auto-chunked lists

// Dynamic shared memory of hs_pass_kernel for a (G, NL) configuration.
__host__ __device__ constexpr size_t hs_pass_smem_bytes(int G, int NL)
{
    return sizeof(float2) * (size_t)G * NL * (1 + kThreads / G);
}

template <int G, int NL, int MODE>
__global__ void __launch_bounds__(kThreads, (NL > 16 ? 1 : 2))
hs_pass_kernel(const PassArgs a)
{
    constexpr int SPW = 32 / G;
    constexpr int NSLOT = kThreads / G;
    constexpr int NV = NL / 2;
    constexpr bool BWD = (MODE & PM_BWD) != 0;
    constexpr bool FWD = (MODE & PM_FWD) != 0;
    constexpr bool WRITE = (MODE & PM_WRITE) != 0;
    extern __shared__ float4 smem4[];

    const int pat = blockIdx.y;
    const int chunk = a.f.chunk_base + blockIdx.x;
    if (a.f.u.status[pat] != 0) return;  // pattern already failed (uniform per CTA)

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane % G, s = lane / G;
    const int slot = warp * SPW + s;
    constexpr int npv = G * NV;    // float4 per table row (np = G * NL)
    float4 *coef_s = smem4;                  // [npv]
    float4 *E_s = smem4 + npv;               // [NSLOT][npv]

    if (BWD) {
        const float4 *cg = reinterpret_cast<const float4 *>(a.coef + (int64_t)pat * a.np);
        for (int k = tid; k < npv; k += kThreads) coef_s[k] = cg[k];
    }
    if (FWD)
        for (int k = tid; k < NSLOT * npv; k += kThreads) E_s[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();

    const float4 *__restrict__ X = reinterpret_cast<const float4 *>(a.gx + (int64_t)pat * a.tab_stride) + g;
    const float4 *__restrict__ Y = reinterpret_cast<const float4 *>(a.gy + (int64_t)pat * a.tab_stride) + g;

    // V = coef * gy[row] (backward), T = sum_p b_p gx[c_p] (forward), per row.
    float vr[NL], vi[NL], tr[NL], ti[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) { vr[k] = 0.f; vi[k] = 0.f; tr[k] = 0.f; ti[k] = 0.f; }

    auto flush = [&](int r) {
        // E_slot += gy[r] * T ; T = 0
        const float4 *yr = Y + (int64_t)r * npv;
        float4 *es = E_s + slot * npv + g;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const float4 q = __ldg(yr + G * j);
            float4 e = es[G * j];
            e.x = fmaf(q.x, tr[2 * j], e.x);
            e.x = fmaf(-q.y, ti[2 * j], e.x);
            e.y = fmaf(q.x, ti[2 * j], e.y);
            e.y = fmaf(q.y, tr[2 * j], e.y);
            e.z = fmaf(q.z, tr[2 * j + 1], e.z);
            e.z = fmaf(-q.w, ti[2 * j + 1], e.z);
            e.w = fmaf(q.z, ti[2 * j + 1], e.w);
            e.w = fmaf(q.w, tr[2 * j + 1], e.w);
            es[G * j] = e;
            tr[2 * j] = 0.f; ti[2 * j] = 0.f; tr[2 * j + 1] = 0.f; ti[2 * j + 1] = 0.f;
        }
    };

    const int64_t begin = (int64_t)chunk * a.chunk_len;
    const int wseg = a.chunk_len / kWarps;
    const int64_t wbegin = begin + (int64_t)warp * wseg;
    int64_t wend = wbegin + wseg;
    if (wend > a.count) wend = a.count;
    const int trips = (wend > wbegin) ? (int)((wend - wbegin + SPW - 1) / SPW) : 0;
    int rcur = -1;

    for (int t = 0; t < trips; ++t) {
        const int64_t i = wbegin + (int64_t)t * SPW + s;
        const bool valid = i < wend;
        int rc = 0;
        float A = 0.f;
        if (valid) { rc = __ldg(a.rc + i); A = __ldg(a.amp + i); }
        const int r = valid ? (rc >> 16) : rcur;
        const int c = valid ? (rc & 0xffff) : 0;
        if (r != rcur && r >= 0) {
            if (FWD && rcur >= 0) flush(rcur);
            if (BWD) {
                const float4 *yr = Y + (int64_t)r * npv;
                const float4 *cs = coef_s + g;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const float4 q = __ldg(yr + G * j);
                    const float4 k4 = cs[G * j];
                    vr[2 * j] = fmaf(k4.x, q.x, -k4.y * q.y);
                    vi[2 * j] = fmaf(k4.x, q.y, k4.y * q.x);
                    vr[2 * j + 1] = fmaf(k4.z, q.z, -k4.w * q.w);
                    vi[2 * j + 1] = fmaf(k4.z, q.w, k4.w * q.z);
                }
            }
            rcur = r;
        }
        float xr[NL], xi[NL];
        const float4 *xc = X + (int64_t)c * npv;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const float4 q = __ldg(xc + G * j);
            xr[2 * j] = q.x; xi[2 * j] = q.y; xr[2 * j + 1] = q.z; xi[2 * j + 1] = q.w;
        }

        float br, bi;
        if (BWD) {
            float s0r = 0.f, s0i = 0.f, s1r = 0.f, s1i = 0.f;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                s0r = fmaf(vr[2 * j], xr[2 * j], s0r);
                s0r = fmaf(-vi[2 * j], xi[2 * j], s0r);
                s0i = fmaf(vr[2 * j], xi[2 * j], s0i);
                s0i = fmaf(vi[2 * j], xr[2 * j], s0i);
                s1r = fmaf(vr[2 * j + 1], xr[2 * j + 1], s1r);
                s1r = fmaf(-vi[2 * j + 1], xi[2 * j + 1], s1r);
                s1i = fmaf(vr[2 * j + 1], xi[2 * j + 1], s1i);
                s1i = fmaf(vi[2 * j + 1], xr[2 * j + 1], s1i);
            }
            float sr = s0r + s1r, si = s0i + s1i;
            // Butterfly over the G lanes of the pixel (a+b == b+a: all lanes
            // end with identical bits).
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                sr += __shfl_xor_sync(0xffffffffu, sr, o);
                si += __shfl_xor_sync(0xffffffffu, si, o);
            }
            // b = A e^{-i arg S} = A conj(S)/|S|; arg(0) = 0 (kernels.py:115-119)
            const float m2 = fmaf(sr, sr, si * si);
            if (m2 > 0.f && m2 < INFINITY) {
                const float inv = A * rsqrtf(m2);
                br = sr * inv;
                bi = -si * inv;
            } else if (sr != 0.f || si != 0.f) {
                const float mx = fmaxf(fabsf(sr), fabsf(si));
                const float xr_ = sr / mx, xi_ = si / mx;
                const float inv = A * rsqrtf(fmaf(xr_, xr_, xi_ * xi_));
                br = xr_ * inv;
                bi = -xi_ * inv;
            } else {
                br = A;
                bi = 0.f;
            }
            if (WRITE && valid && g == 0) {
                const int64_t di = a.dst ? (int64_t)a.dst[i] : i + a.idx_base;
                if (di >= 0) {
                    hs_store_phase(a.phase_out, a.phase_out32, (int64_t)pat * a.phase_stride + di, sr, si);
                    if (a.raster)
                        a.raster[(int64_t)pat * a.side * a.side + (int64_t)(rc >> 16) * a.side + (rc & 0xffff)] =
                            hs_gray_linear(hs_phase_f64(sr, si));
                }
            }
        } else {
            double sn = 0.0, cs = 1.0;
            if (valid) {
                const int64_t di = a.dst ? (int64_t)a.dst[i] : i + a.idx_base;
                if (di >= 0) sincos(a.phase_in[(int64_t)pat * a.phase_stride + di], &sn, &cs);
            }
            br = A * (float)cs;
            bi = -A * (float)sn;
        }

        if (FWD) {
#pragma unroll
            for (int k = 0; k < NL; ++k) {
                tr[k] = fmaf(br, xr[k], tr[k]);
                tr[k] = fmaf(-bi, xi[k], tr[k]);
                ti[k] = fmaf(br, xi[k], ti[k]);
                ti[k] = fmaf(bi, xr[k], ti[k]);
            }
        }
    }

    if (FWD) {
        if (rcur >= 0) flush(rcur);
        __syncthreads();
        // per-chunk partial: slots folded in slot order (fixed)
        const float2 *E2 = reinterpret_cast<const float2 *>(E_s);
        float2 *out = a.f.partials + (int64_t)pat * a.f.part_stride + (int64_t)chunk * a.np;
        for (int k = tid; k < a.np; k += kThreads) {
            float sx = 0.f, sy = 0.f;
#pragma unroll 8
            for (int q = 0; q < NSLOT; ++q) {
                const float2 v = E2[q * a.np + k];
                sx += v.x;
                sy += v.y;
            }
            out[k] = make_float2(sx, sy);
        }
        if (a.f.u.act != ACT_NONE) {
            __syncthreads();
            hs_fold(a.f, pat, chunk, reinterpret_cast<char *>(E_s));
        }
    }
}

// Kernel selection (instantiated per G in hs_pass_g*.cu).
typedef void (*PassFn)(PassArgs);

template <int G, int NL>
PassFn hs_pass_fn(int mode)
{
    switch (mode) {
    case PM_BWD | PM_WRITE: return hs_pass_kernel<G, NL, PM_BWD | PM_WRITE>;
    case PM_FWD: return hs_pass_kernel<G, NL, PM_FWD>;
    case PM_BWD | PM_FWD: return hs_pass_kernel<G, NL, PM_BWD | PM_FWD>;
    case PM_BWD | PM_FWD | PM_WRITE: return hs_pass_kernel<G, NL, PM_BWD | PM_FWD | PM_WRITE>;
    default: return nullptr;
    }
}

PassFn hs_select_g1(int nl, int mode);
PassFn hs_select_g2(int nl, int mode);
PassFn hs_select_g4(int nl, int mode);
PassFn hs_select_g8(int nl, int mode);
PassFn hs_select_g16(int nl, int mode);
PassFn hs_select_g32(int nl, int mode);

#define HS_DEFINE_SELECT(GV)                                  \
    PassFn hs_select_g##GV(int nl, int mode)                  \
    {                                                         \
        switch (nl) {                                         \
        case 4: return hs_pass_fn<GV, 4>(mode);               \
        case 8: return hs_pass_fn<GV, 8>(mode);               \
        case 10: return hs_pass_fn<GV, 10>(mode);             \
        case 12: return hs_pass_fn<GV, 12>(mode);             \
        case 14: return hs_pass_fn<GV, 14>(mode);             \
        case 16: return hs_pass_fn<GV, 16>(mode);             \
        default: return nullptr;                              \
        }                                                     \
    }

// ---------------------------------------------------------------------------
// Row-sharded passes (paper_2003_05293_b200/distributed.py): the chunk range of
// a rank is folded group by group (same order and precision as hs_fold's first
// level), the group partials of all ranks are exchanged, and every rank runs
// the second level + update on the identical group sequence.
static __global__ void hs_group_fold_kernel(FoldArgs a, int g_lo)
{
    const int pat = blockIdx.y, grp = g_lo + blockIdx.x, np = a.np;
    const int c0 = grp * kGroup, c1 = min(c0 + kGroup, a.nchunks);
    const float2 *part = a.partials + (int64_t)pat * a.part_stride;
    double2 *gp = a.gpart + (int64_t)pat * a.gpart_stride;
    for (int k = threadIdx.x; k < np; k += blockDim.x) {
        double sx = 0.0, sy = 0.0;
        for (int c = c0; c < c1; ++c) {
            const float2 v = part[(int64_t)c * np + k];
            sx += (double)v.x;
            sy += (double)v.y;
        }
        gp[(int64_t)grp * np + k] = make_double2(sx, sy);
    }
}

static __global__ void __launch_bounds__(kThreads) hs_fold_update_kernel(FoldArgs a, int ngroups)
{
    __shared__ double dbuf[kThreads];
    __shared__ int ibuf[kThreads];
    extern __shared__ double2 Eu[];          // [np] fields + [2 np] scratch
    const int pat = blockIdx.x, np = a.np;
    if (a.u.status[pat] != 0) return;
    const double2 *gp = a.gpart + (int64_t)pat * a.gpart_stride;
    for (int k = threadIdx.x; k < np; k += kThreads) {
        double sx = 0.0, sy = 0.0;
        for (int g = 0; g < ngroups; ++g) {
            const double2 v = gp[(int64_t)g * np + k];
            sx += v.x;
            sy += v.y;
        }
        Eu[k] = make_double2(sx, sy);
    }
    __syncthreads();
    hs_update(a.u, pat, Eu, reinterpret_cast<double *>(Eu + np), dbuf, ibuf);
}

}  // namespace hs
