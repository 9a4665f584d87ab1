// hs_tile.cuh -- full-range fused pass as two register-blocked complex GEMMs.
//
// A CTA owns one 64-row x 32-column tile of the SLM grid (all of its pixels,
// zero-amplitude outside the aperture) for one pattern.  With the spot
// phasors of the tile's columns X[k][c] = gx[c0+c][k] and rows
// V[k][r] = coef_k gy[r0+r][k] staged in shared memory:
//
//   backward  S[r][c] = sum_k V[k][r] X[k][c]        (kernels.py:99-119)
//             b[r][c] = A[r][c] conj(S)/|S|           (forward input, kernels.py:136-137)
//   forward   T[r][k] = sum_c b[r][c] X[k][c]         (kernels.py:122-144, per row)
//             E_k    += sum_r gy[r0+r][k] T[r][k]
//
// Both products are complex GEMMs with K = spots (backward) and K = 32
// columns (forward); each thread keeps a 4x2 (backward) / 4xNS (forward)
// register tile, so shared-memory traffic is a small fraction of the FFMA
// work.  The CTA's per-spot partial is folded by the same fixed-order
// two-level tree as the pass kernel (hs_fold).
#pragma once

#include "hs_kernels.cuh"

namespace hs {

constexpr int kTileR = 64;        // tile rows
constexpr int kTileC = 32;        // tile columns
constexpr int kXS = kTileC + 1;   // X row stride (complex): conflict-free column reads
constexpr int kVS = kTileR + 2;   // V row stride (complex), keeps 16-B alignment
constexpr int kBS = kTileR + 4;   // b row stride (complex), 16-B aligned

struct TileArgs {
    const int32_t *tiles;     // packed (r0 << 16) | c0 per tile
    int32_t side;
    int32_t np;               // 16 * NS
    int64_t tab_stride;       // side * np
    const float2 *gx, *gy;    // [B][side][np]
    const float2 *coef;       // [B][np]
    const float *amp_img;     // [side][side], 0 outside the aperture
    const int32_t *idx_img;   // [side][side] storage index, -1 outside
    double *phase_out;        // [B][phase_stride] (WRITE)
    unsigned char *raster;    // [B][side][side] SLM gray raster (WRITE, nullable)
    int64_t phase_stride;
    FoldArgs f;
};

// Second region: V [np][kVS] during the backward product; afterwards b
// [kTileC][kBS] + the row-group fold [16][np] (+ hs_fold scratch).
__host__ __device__ constexpr int hs_tile_region2(int NS)
{
    return (16 * NS * kVS > kTileC * kBS + 16 * 16 * NS) ? 16 * NS * kVS : kTileC * kBS + 16 * 16 * NS;
}

__host__ __device__ constexpr size_t hs_tile_smem_bytes(int NS)
{
    return sizeof(float2) * ((size_t)16 * NS * kXS + hs_tile_region2(NS));
}

template <int NS, bool WRITE>
__global__ void __launch_bounds__(kThreads, 2) hs_tile_kernel(const TileArgs a)
{
    constexpr int NP = 16 * NS;
    extern __shared__ float2 sm2[];
    float2 *Xs = sm2;                     // [NP][kXS]
    float2 *Vs = Xs + NP * kXS;           // [NP][kVS]
    float2 *Bs = Vs;                      // [kTileC][kBS]   (after backward)
    float2 *Rs = Vs + kTileC * kBS;       // [16][NP]        (after forward)

    const int pat = blockIdx.y;
    const int tile = a.f.chunk_base + blockIdx.x;
    if (a.f.u.status[pat] != 0) return;
    const int tid = threadIdx.x;
    const int packed = __ldg(a.tiles + tile);
    const int r0 = packed >> 16, c0 = packed & 0xffff;
    const float2 *gx = a.gx + (int64_t)pat * a.tab_stride;
    const float2 *gy = a.gy + (int64_t)pat * a.tab_stride;
    const float2 *cf = a.coef + (int64_t)pat * NP;

    // ---- stage X[k][c] and V[k][r] = coef_k gy[r][k] (coalesced over k)
    for (int idx = tid; idx < NP * kTileC; idx += kThreads) {
        const int c = idx / NP, k = idx % NP;
        const int cc = min(c0 + c, a.side - 1);
        Xs[k * kXS + c] = __ldg(gx + (int64_t)cc * NP + k);
    }
    for (int idx = tid; idx < NP * kTileR; idx += kThreads) {
        const int r = idx / NP, k = idx % NP;
        const int rr = min(r0 + r, a.side - 1);
        const float2 q = __ldg(gy + (int64_t)rr * NP + k);
        const float2 w = __ldg(cf + k);
        Vs[k * kVS + r] = make_float2(fmaf(w.x, q.x, -w.y * q.y), fmaf(w.x, q.y, w.y * q.x));
    }
    __syncthreads();

    // ---- backward: warp (wr, wc) covers rows 16wr.., cols 16wc..;
    //      lane (lr, lc) holds rows 4lr..4lr+3, cols 2lc, 2lc+1 of that block.
    const int lane = tid & 31, warp = tid >> 5;
    const int rb = 16 * (warp >> 1) + 4 * (lane >> 3);
    const int cb = 16 * (warp & 1) + 2 * (lane & 7);
    float sr[4][2], si[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) { sr[i][j] = 0.f; si[i][j] = 0.f; }
#pragma unroll 4
    for (int k = 0; k < NP; ++k) {
        const float4 v01 = *reinterpret_cast<const float4 *>(Vs + k * kVS + rb);
        const float4 v23 = *reinterpret_cast<const float4 *>(Vs + k * kVS + rb + 2);
        const float2 x0 = Xs[k * kXS + cb];
        const float2 x1 = Xs[k * kXS + cb + 1];
        const float vr[4] = {v01.x, v01.z, v23.x, v23.z};
        const float vi[4] = {v01.y, v01.w, v23.y, v23.w};
        const float xr[2] = {x0.x, x1.x};
        const float xi[2] = {x0.y, x1.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                sr[i][j] = fmaf(vr[i], xr[j], sr[i][j]);
                sr[i][j] = fmaf(-vi[i], xi[j], sr[i][j]);
                si[i][j] = fmaf(vr[i], xi[j], si[i][j]);
                si[i][j] = fmaf(vi[i], xr[j], si[i][j]);
            }
    }

    // ---- b = A conj(S)/|S| (arg(0) = 0); optional phase write
    float br[4][2], bi[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int r = r0 + rb + i, c = c0 + cb + j;
            const bool in = (r < a.side) && (c < a.side);
            const int64_t gidx = (int64_t)r * a.side + c;
            const float A = in ? __ldg(a.amp_img + gidx) : 0.f;
            const float x = sr[i][j], y = si[i][j];
            const float m2 = fmaf(x, x, y * y);
            if (m2 > 0.f && m2 < INFINITY) {
                const float inv = A * rsqrtf(m2);
                br[i][j] = x * inv;
                bi[i][j] = -y * inv;
            } else if (x != 0.f || y != 0.f) {
                const float mx = fmaxf(fabsf(x), fabsf(y));
                const float xr_ = x / mx, xi_ = y / mx;
                const float inv = A * rsqrtf(fmaf(xr_, xr_, xi_ * xi_));
                br[i][j] = xr_ * inv;
                bi[i][j] = -xi_ * inv;
            } else {
                br[i][j] = A;
                bi[i][j] = 0.f;
            }
            if (WRITE && in) {
                const int32_t di = __ldg(a.idx_img + gidx);
                if (di >= 0) {
                    double ph = 0.0;
                    if (x != 0.f || y != 0.f) {
                        ph = (double)atan2f(y, x);
                        if (ph >= kPi) ph -= kTwoPi;       // pi -> -pi convention
                        else if (ph < -kPi) ph += kTwoPi;  // fp32 -pi lies below fp64 -pi
                    }
                    a.phase_out[(int64_t)pat * a.phase_stride + di] = ph;
                    if (a.raster) a.raster[(int64_t)pat * a.side * a.side + gidx] = hs_gray_linear(ph);
                }
            }
        }
    __syncthreads();  // V no longer read: reuse its space for b
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        float4 *dst = reinterpret_cast<float4 *>(Bs + (cb + j) * kBS + rb);
        dst[0] = make_float4(br[0][j], bi[0][j], br[1][j], bi[1][j]);
        dst[1] = make_float4(br[2][j], bi[2][j], br[3][j], bi[3][j]);
    }
    __syncthreads();

    // ---- forward: thread (rg, sg) holds rows 4rg..4rg+3 x spots sg + 16j
    const int rg = tid >> 4, sg = tid & 15;
    float tr[4][NS], ti[4][NS];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NS; ++j) { tr[i][j] = 0.f; ti[i][j] = 0.f; }
#pragma unroll 2
    for (int c = 0; c < kTileC; ++c) {
        const float4 b01 = *reinterpret_cast<const float4 *>(Bs + c * kBS + 4 * rg);
        const float4 b23 = *reinterpret_cast<const float4 *>(Bs + c * kBS + 4 * rg + 2);
        const float bre[4] = {b01.x, b01.z, b23.x, b23.z};
        const float bim[4] = {b01.y, b01.w, b23.y, b23.w};
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            const float2 x = Xs[(sg + 16 * j) * kXS + c];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                tr[i][j] = fmaf(bre[i], x.x, tr[i][j]);
                tr[i][j] = fmaf(-bim[i], x.y, tr[i][j]);
                ti[i][j] = fmaf(bre[i], x.y, ti[i][j]);
                ti[i][j] = fmaf(bim[i], x.x, ti[i][j]);
            }
        }
    }
    // E_k += sum_i gy[r][k] T[i][k], then fold the 16 row groups in order
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        const int k = sg + 16 * j;
        float er = 0.f, ei = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int rr = min(r0 + 4 * rg + i, a.side - 1);
            const float2 q = __ldg(gy + (int64_t)rr * NP + k);
            er = fmaf(q.x, tr[i][j], er);
            er = fmaf(-q.y, ti[i][j], er);
            ei = fmaf(q.x, ti[i][j], ei);
            ei = fmaf(q.y, tr[i][j], ei);
        }
        Rs[rg * NP + k] = make_float2(er, ei);
    }
    __syncthreads();
    float2 *out = a.f.partials + (int64_t)pat * a.f.part_stride + (int64_t)tile * NP;
    for (int k = tid; k < NP; k += kThreads) {
        float x = 0.f, y = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float2 v = Rs[q * NP + k];
            x += v.x;
            y += v.y;
        }
        out[k] = make_float2(x, y);
    }
    if (a.f.u.act != ACT_NONE) {
        __syncthreads();
        hs_fold(a.f, pat, tile, reinterpret_cast<char *>(Vs));
    }
}

typedef void (*TileFn)(TileArgs);
TileFn hs_select_tile(int ns, bool write);

}  // namespace hs
