// hs_tilek.cuh -- full-range fused pass for large spot counts (n > 128).
//
// Same 64 x 64-pixel tiles and GEMM formulation as hs_tile.cuh
// (backward kernels.py:99-119, forward kernels.py:122-144), with the spot
// dimension streamed through shared memory in chunks of kKC spots so any
// n <= 1024 fits (config 4: N = 1000):
//
//   backward  for each spot chunk: stage X[k][c] = gx[c0+c][k] and
//             V[k][r] = coef_k gy[r0+r][k], accumulate S[r][c] (4 x 4 per
//             thread, FFMA2 complex MACs)
//   b         = A conj(S)/|S| into shared memory (+ the phase on the last pass)
//   forward   for each spot chunk: stage X again, T[r][k] = sum_c b[r][c] X[k][c]
//             (2 rows x 8 spots per thread), E_k = sum_r gy[r0+r][k] T[r][k]
//             summed over the 32 row groups in order -> the tile's partial
//
// ~101 KB of shared memory: two CTAs per SM, so one CTA's chunk staging
// overlaps the other's math.  Partials are folded by the fixed-order tree
// (hs_fold), so results are deterministic and batch-invariant.
#pragma once

#include "hs_f2.cuh"
#include "hs_kernels.cuh"
#include "hs_tile.cuh"

namespace hs {

constexpr int kKC = 64;  // spots per chunk

__host__ __device__ constexpr size_t hs_tilek_smem_bytes()
{
    // X chunk [kKC][kXS] + V chunk [kKC][kVS] (later row-group partials) + b [64][kBS]
    return sizeof(float2) * ((size_t)kKC * kXS + (size_t)kKC * kVS + (size_t)kTileC * kBS);
}

template <bool WRITE>
__global__ void __launch_bounds__(kThreads, 2) hs_tilek_kernel(const TileArgs a)
{
    extern __shared__ float2 smk[];
    float2 *Xs = smk;                  // [kKC][kXS]
    float2 *Vs = Xs + kKC * kXS;       // [kKC][kVS]   (forward: row-group partials [32][kKC])
    float2 *Bs = Vs + kKC * kVS;       // [kTileC][kBS]
    float2 *Rs = Vs;

    hs_pdl_launch_next();
    hs_pdl_wait_prev();  // coef / status of the previous pass
    const int pat = blockIdx.y;
    const int tile = a.f.chunk_base + blockIdx.x;
    if (a.f.u.status[pat] != 0) return;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int packed = __ldg(a.tiles + tile);
    const int r0 = packed >> 16, c0 = packed & 0xffff;
    const float2 *gx = a.gx + (int64_t)pat * a.tab_stride;
    const float2 *gy = a.gy + (int64_t)pat * a.tab_stride;
    const float2 *cf = a.coef + (int64_t)pat * a.np;
    const int nchunk = (a.np + kKC - 1) / kKC;

    // stage X[k][c] for spots k0 .. k0 + kKC (zeros past np); warp w takes
    // columns w + 8 i, lane l spots l and l + 32 (coalesced table rows)
    auto stage_x = [&](int k0) {
        float2 v[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 *src = gx + (int64_t)min(c0 + warp + 8 * i, a.side - 1) * a.np + k0;
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const int k = lane + 32 * m;
                v[i][m] = (k0 + k < a.np) ? __ldg(src + k) : make_float2(0.f, 0.f);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int m = 0; m < 2; ++m) Xs[(lane + 32 * m) * kXS + warp + 8 * i] = v[i][m];
    };
    auto stage_v = [&](int k0) {
        float2 v[8][2], w[2];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const int k = k0 + lane + 32 * m;
            w[m] = (k < a.np) ? __ldg(cf + k) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 *src = gy + (int64_t)min(r0 + warp + 8 * i, a.side - 1) * a.np + k0;
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const int k = lane + 32 * m;
                v[i][m] = (k0 + k < a.np) ? __ldg(src + k) : make_float2(0.f, 0.f);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const float2 q = v[i][m];
                Vs[(lane + 32 * m) * kVS + warp + 8 * i] =
                    make_float2(fmaf(w[m].x, q.x, -w[m].y * q.y), fmaf(w[m].x, q.y, w[m].y * q.x));
            }
    };

    // ---- backward over spot chunks: thread (tr, tc) holds rows 4 tr + i, columns tc + 16 j
    const int tr = tid >> 4, tc = tid & 15;
    f2x sacc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sacc[i][j] = 0ull;
    const f2x *X2 = reinterpret_cast<const f2x *>(Xs);
    for (int ch = 0; ch < nchunk; ++ch) {
        stage_x(ch * kKC);
        stage_v(ch * kKC);
        __syncthreads();
#pragma unroll 16
        for (int k = 0; k < kKC; ++k) {
            const float4 v01 = *reinterpret_cast<const float4 *>(Vs + k * kVS + 4 * tr);
            const float4 v23 = *reinterpret_cast<const float4 *>(Vs + k * kVS + 4 * tr + 2);
            f2x x[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = X2[k * kXS + tc + 16 * j];
            const float vr[4] = {v01.x, v01.z, v23.x, v23.z};
            const float vi[4] = {v01.y, v01.w, v23.y, v23.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) f2_cmac(sacc[i][j], vr[i], vi[i], x[j]);
        }
        __syncthreads();
    }

    // ---- b = A conj(S)/|S| into Bs[c][r]; optional phase write
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = r0 + 4 * tr + i, c = c0 + tc + 16 * j;
            const bool in = (r < a.side) && (c < a.side);
            const int64_t gidx = (int64_t)r * a.side + c;
            const float A = in ? __ldg(a.amp_img + gidx) : 0.f;
            const float x = f2_lo(sacc[i][j]), y = f2_hi(sacc[i][j]);
            float br, bi;
            hs_bvec_exact(x, y, A, br, bi);
            Bs[(tc + 16 * j) * kBS + 4 * tr + i] = make_float2(br, bi);
            if (WRITE && in) {
                const int32_t di = __ldg(a.idx_img + gidx);
                if (di >= 0) {
                    hs_store_phase(a.phase_out, a.phase_out32, (int64_t)pat * a.phase_stride + di, x, y);
                    if (a.raster)
                        a.raster[(int64_t)pat * a.side * a.side + gidx] = hs_gray_linear(hs_phase_f64(x, y));
                }
            }
        }

    // ---- forward over spot chunks: thread (rg, sg) rows 2 rg, 2 rg + 1 x spots sg + 8 j
    const int rg = tid >> 3, sg = tid & 7;
    const int ra = min(r0 + 2 * rg, a.side - 1), rb = min(r0 + 2 * rg + 1, a.side - 1);
    float2 *out = a.f.partials + (int64_t)pat * a.f.part_stride + (int64_t)tile * a.np;
    for (int ch = 0; ch < nchunk; ++ch) {
        const int k0 = ch * kKC;
        stage_x(k0);
        __syncthreads();  // X staged (and, on the first chunk, b complete)
        f2x t0[8], t1[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) t0[j] = t1[j] = 0ull;
#pragma unroll 16
        for (int c = 0; c < kTileC; ++c) {
            const float4 b = *reinterpret_cast<const float4 *>(Bs + c * kBS + 2 * rg);
            f2x x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = X2[(sg + 8 * j) * kXS + c];
#pragma unroll
            for (int j = 0; j < 8; ++j) f2_cmac(t0[j], b.x, b.y, x[j]);
#pragma unroll
            for (int j = 0; j < 8; ++j) f2_cmac(t1[j], b.z, b.w, x[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int k = k0 + sg + 8 * j;
            f2x e = 0ull;
            if (k < a.np) {
                const float2 qa = __ldg(gy + (int64_t)ra * a.np + k);
                const float2 qb = __ldg(gy + (int64_t)rb * a.np + k);
                f2_cmac(e, qa.x, qa.y, t0[j]);
                f2_cmac(e, qb.x, qb.y, t1[j]);
            }
            reinterpret_cast<f2x *>(Rs)[rg * kKC + sg + 8 * j] = e;
        }
        __syncthreads();
        for (int k = tid; k < kKC; k += kThreads) {
            float x = 0.f, y = 0.f;
#pragma unroll 8
            for (int q = 0; q < 32; ++q) {
                const float2 v = Rs[q * kKC + k];
                x += v.x;
                y += v.y;
            }
            if (k0 + k < a.np) out[k0 + k] = make_float2(x, y);
        }
        __syncthreads();  // Rs and Xs free for the next chunk
    }
    if (a.f.u.act != ACT_NONE) hs_fold(a.f, pat, tile, reinterpret_cast<char *>(Vs));
}

typedef void (*TileKFn)(TileArgs);
TileKFn hs_select_tilek(bool write);

}  // namespace hs
