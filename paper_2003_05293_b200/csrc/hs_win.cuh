// hs_win.cuh -- compressed-window fused pass (solver iterations 1..I-2).
//
// Window pixels are a random 1/16 subset of the aperture (storage-order
// window, solvers.py:212-222), listed sorted by (row, col).  A pixel needs
// the gx row of its own column from L2, so this pass is latency-bound; the
// kernel is shaped for memory-level parallelism instead of register reuse:
//
//   * G = 16 lanes per pixel, NL spots per lane (n = g + 16 j), so the
//     per-lane state (V, T, E, gx row and the prefetched next gx row) fits
//     in ~100 registers;
//   * the next pixel's gx row is loaded one trip ahead (software pipeline);
//   * per-row V = coef * gy[row] and T = sum b gx live in registers as in the
//     row-run kernel; E accumulates in registers and is folded across the
//     warp's two slots by shuffle and across warps in a fixed order.
//
// Arithmetic per pixel-spot pair is identical to hs_pass_kernel:
// backward (kernels.py:99-119) + forward (kernels.py:122-144).
#pragma once

#include "hs_kernels.cuh"

namespace hs {

constexpr int kMaxCpc = 4;  // logical chunks per CTA (divides kGroup)

__host__ __device__ constexpr size_t hs_win_smem_bytes(int NL)
{
    return sizeof(float2) * (size_t)16 * NL * (1 + kMaxCpc * kWarps);
}

// One CTA streams `cpc` consecutive logical chunks (a.cpc) of one pattern.
// Each logical chunk keeps its own fixed warp segmentation and its own
// partial, so results do not depend on cpc; the gx prefetch pipeline runs
// across chunk boundaries.
template <int NL, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) hs_win_kernel(const PassArgs a)
{
    constexpr int G = 16;
    constexpr int SPW = 32 / G;
    constexpr int NP = G * NL;
    extern __shared__ float2 smw[];
    float2 *coef_s = smw;           // [NP]
    float2 *Ew = smw + NP;          // [cpc][kWarps][NP]

    const int pat = blockIdx.y;
    if (a.f.u.status[pat] != 0) return;
    const int q0 = a.f.chunk_base + blockIdx.x * a.cpc;
    const int nq = min(a.cpc, a.f.chunk_end - q0);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane & (G - 1), s = lane / G;

    for (int k = tid; k < NP; k += kThreads) coef_s[k] = a.coef[(int64_t)pat * NP + k];
    __syncthreads();

    const float2 *__restrict__ X = a.gx + (int64_t)pat * a.tab_stride + g;
    const float2 *__restrict__ Y = a.gy + (int64_t)pat * a.tab_stride + g;
    const int wseg = a.chunk_len / kWarps;
    const int tf = wseg / SPW;                // trips per logical chunk
    const int total = nq * tf;
    const int64_t wbase = (int64_t)q0 * a.chunk_len + (int64_t)warp * wseg + s;

    float vr[NL], vi[NL], tr[NL], ti[NL], er[NL], ei[NL], xr[NL], xi[NL], nr[NL], ni[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        vr[j] = vi[j] = tr[j] = ti[j] = er[j] = ei[j] = 0.f;
        xr[j] = xi[j] = nr[j] = ni[j] = 0.f;
    }
    // Entry stream (runs two trips ahead of the compute): chunk counter qe,
    // trip-in-chunk te and list index ie advance incrementally.
    int qe = 0, te = 0;
    int64_t ie = wbase;
    const int64_t wrap = (int64_t)a.chunk_len - (int64_t)wseg;
    auto next_entry = [&](int &rc, float &A) {
        rc = -1;
        A = 0.f;
        if (qe < nq && ie < a.count) {
            rc = __ldg(a.rc + ie);
            A = __ldg(a.amp + ie);
        }
        ie += SPW;
        if (++te == tf) {
            te = 0;
            ++qe;
            ie += wrap;
        }
    };
    auto load_x = [&](int rc, float (&dr)[NL], float (&di)[NL]) {
        const float2 *xc = X + (rc < 0 ? 0 : (rc & 0xffff)) * NP;
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const float2 q = __ldg(xc + G * j);
            dr[j] = q.x;
            di[j] = q.y;
        }
    };
    auto flush = [&](int r) {  // E += gy[r] * T ; T = 0
        const float2 *yr = Y + r * NP;
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const float2 q = __ldg(yr + G * j);
            er[j] = fmaf(q.x, tr[j], er[j]);
            er[j] = fmaf(-q.y, ti[j], er[j]);
            ei[j] = fmaf(q.x, ti[j], ei[j]);
            ei[j] = fmaf(q.y, tr[j], ei[j]);
            tr[j] = 0.f;
            ti[j] = 0.f;
        }
    };

    int rc_c, rc_n;
    float A_c, A_n;
    next_entry(rc_c, A_c);
    next_entry(rc_n, A_n);
    load_x(rc_c, xr, xi);
    int rcur = -1, tc = 0, qc = 0;

    // One trip: prefetch the next pixel's gx row into (pr, pi), compute the
    // current pixel from (cr, ci).  Called with the two register sets
    // swapped on alternate trips (no copies).
    auto trip = [&](float (&cr)[NL], float (&ci)[NL], float (&pr)[NL], float (&pi)[NL]) {
        load_x(rc_n, pr, pi);
        int rc_nn;
        float A_nn;
        next_entry(rc_nn, A_nn);

        const int r = rc_c < 0 ? rcur : (rc_c >> 16);
        if (r != rcur && r >= 0) {
            if (rcur >= 0) flush(rcur);
            const float2 *yr = Y + r * NP;
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                const float2 q = __ldg(yr + G * j);
                const float2 w = coef_s[g + G * j];
                vr[j] = fmaf(w.x, q.x, -w.y * q.y);
                vi[j] = fmaf(w.x, q.y, w.y * q.x);
            }
            rcur = r;
        }
        float s0r = 0.f, s0i = 0.f, s1r = 0.f, s1i = 0.f;
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            if (j & 1) {
                s1r = fmaf(vr[j], cr[j], s1r);
                s1r = fmaf(-vi[j], ci[j], s1r);
                s1i = fmaf(vr[j], ci[j], s1i);
                s1i = fmaf(vi[j], cr[j], s1i);
            } else {
                s0r = fmaf(vr[j], cr[j], s0r);
                s0r = fmaf(-vi[j], ci[j], s0r);
                s0i = fmaf(vr[j], ci[j], s0i);
                s0i = fmaf(vi[j], cr[j], s0i);
            }
        }
        float sr = s0r + s1r, si = s0i + s1i;
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            sr += __shfl_xor_sync(0xffffffffu, sr, o);
            si += __shfl_xor_sync(0xffffffffu, si, o);
        }
        float br, bi;
        const float m2 = fmaf(sr, sr, si * si);
        if (m2 > 0.f && m2 < INFINITY) {
            const float inv = A_c * rsqrtf(m2);
            br = sr * inv;
            bi = -si * inv;
        } else if (sr != 0.f || si != 0.f) {
            const float mx = fmaxf(fabsf(sr), fabsf(si));
            const float xr_ = sr / mx, xi_ = si / mx;
            const float inv = A_c * rsqrtf(fmaf(xr_, xr_, xi_ * xi_));
            br = xr_ * inv;
            bi = -xi_ * inv;
        } else {
            br = A_c;
            bi = 0.f;
        }
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            tr[j] = fmaf(br, cr[j], tr[j]);
            tr[j] = fmaf(-bi, ci[j], tr[j]);
            ti[j] = fmaf(br, ci[j], ti[j]);
            ti[j] = fmaf(bi, cr[j], ti[j]);
        }
        rc_c = rc_n;
        A_c = A_n;
        rc_n = rc_nn;
        A_n = A_nn;

        if (++tc == tf) {
            // end of logical chunk qc: its E, slots folded by one symmetric
            // add, stored per warp; state restarts for the next chunk.
            if (rcur >= 0) flush(rcur);
            rcur = -1;
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                const float ex = er[j] + __shfl_xor_sync(0xffffffffu, er[j], 16);
                const float ey = ei[j] + __shfl_xor_sync(0xffffffffu, ei[j], 16);
                if (s == 0) Ew[(qc * kWarps + warp) * NP + g + G * j] = make_float2(ex, ey);
                er[j] = 0.f;
                ei[j] = 0.f;
            }
            tc = 0;
            ++qc;
        }
    };

    int T = 0;
    for (; T + 1 < total; T += 2) {
        trip(xr, xi, nr, ni);
        trip(nr, ni, xr, xi);
    }
    if (T < total) trip(xr, xi, nr, ni);
    __syncthreads();
    for (int k = tid; k < nq * NP; k += kThreads) {
        const int q = k / NP, n = k - q * NP;
        float x = 0.f, y = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float2 v = Ew[(q * kWarps + w) * NP + n];
            x += v.x;
            y += v.y;
        }
        a.f.partials[(int64_t)pat * a.f.part_stride + (int64_t)(q0 + q) * NP + n] = make_float2(x, y);
    }
    if (a.f.u.act != ACT_NONE) {
        __syncthreads();
        hs_fold(a.f, pat, q0, reinterpret_cast<char *>(smw), nq);
    }
}

typedef void (*WinFn)(PassArgs);
WinFn hs_select_win(int nl, int minb = 2);

}  // namespace hs
