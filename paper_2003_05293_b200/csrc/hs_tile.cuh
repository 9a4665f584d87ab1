// hs_tile.cuh -- full-range fused pass as two register-blocked complex GEMMs.
//
// A CTA owns one 64 x 64-pixel tile of the SLM grid (all of its pixels,
// zero amplitude outside the aperture) for one pattern.  With the tile's
// column phasors X[k][c] = gx[c0+c][k] and row phasors
// V[k][r] = coef_k gy[r0+r][k] staged in shared memory:
//
//   backward  S[r][c] = sum_{k<n} V[k][r] X[k][c]      (kernels.py:99-119)
//             b[r][c] = A[r][c] conj(S)/|S|            (kernels.py:136-137)
//   forward   T[r][k] = sum_c b[r][c] X[k][c]          (kernels.py:122-144, per row)
//             E_k    += sum_r gy[r0+r][k] T[r][k]
//
// Register tiles: backward 4 rows x 4 columns per thread (6 shared loads per
// 64 FFMA; each V value feeds 8 consecutive FFMAs, so the register-reuse
// cache keeps the FFMAs at two register reads -- 3-read FFMAs issue at 2/3
// rate, tools/ffma_probe.cu); forward 2 rows x SPT spots per thread
// (spots sg + 8 j, KP = 8 SPT >= n).  The backward runs over the n real spots
// only (rounded to even), the forward over KP = 8 ceil(n / 8) -- not the
// table's 16-spot padding.  Shared memory ~110 KB at n = 100: two CTAs per
// SM, so one CTA's staging overlaps the other's math.  The CTA's per-spot
// partial is folded by the fixed-order two-level tree (hs_fold).
#pragma once

#include "hs_f2.cuh"
#include "hs_kernels.cuh"

namespace hs {

constexpr int kTileR = 64;   // tile rows
constexpr int kTileC = 64;   // tile columns
constexpr int kXS = kTileC + 1;  // X row stride (complex): conflict-free spot-strided reads
constexpr int kVS = kTileR + 2;  // V row stride (complex): 16-B rows, 2-way staging stores
constexpr int kBS = kTileR + 2;  // b row stride ([c][r], complex)

struct TileArgs {
    const int32_t *tiles;     // packed (r0 << 16) | c0 per tile
    int32_t side;
    int32_t np;               // table row stride (spots, 16-padded)
    int32_t n;                // real spots
    int64_t tab_stride;       // side * np
    const float2 *gx, *gy;    // [B][side][np]
    const float *gyp;         // [B][gyp_stride] gy operand planes of the tcgen05 pass (hs_umma.cuh)
    int64_t gyp_stride;
    const float2 *coef;       // [B][np]
    const float *amp_img;     // [side][side], 0 outside the aperture
    const int32_t *idx_img;   // [side][side] storage index, -1 outside
    double *phase_out;        // [B][phase_stride] (WRITE)
    float *phase_out32;       // the same as 4-byte phase codes (WRITE; replaces phase_out)
    unsigned char *raster;    // [B][side][side] SLM gray raster (WRITE, nullable)
    int64_t phase_stride;
    FoldArgs f;
    unsigned long long *trace;  // timing probe of one CTA (hs_umma_kernel, HS_UMMA_TRACE), normally null
};

__host__ __device__ constexpr int hs_tile_kb(int n) { return (n + 1) & ~1; }

// region 1: X [KP][kXS]; region 2: V [kb][kVS], later b [64][kBS], later the
// row-group partials [32][KP] and the hs_fold scratch.
__host__ __device__ constexpr size_t hs_tile_smem_bytes(int spt, int n)
{
    return sizeof(float2) * ((size_t)8 * spt * kXS + (size_t)(hs_tile_kb(n) > kTileC ? hs_tile_kb(n) : kTileC) * kVS);
}

__device__ __forceinline__ void hs_bvec_exact(float x, float y, float A, float &br, float &bi)
{
    const float m2 = fmaf(x, x, y * y);
    if (m2 > 0.f && m2 < INFINITY) {
        const float inv = A * rsqrtf(m2);
        br = x * inv;
        bi = -y * inv;
    } else if (x != 0.f || y != 0.f) {
        const float mx = fmaxf(fabsf(x), fabsf(y));
        const float xr = x / mx, xi = y / mx;
        const float inv = A * rsqrtf(fmaf(xr, xr, xi * xi));
        br = xr * inv;
        bi = -xi * inv;
    } else {
        br = A;
        bi = 0.f;
    }
}

template <int SPT, bool WRITE>
__global__ void __launch_bounds__(kThreads, 2) hs_tile_kernel(const TileArgs a)
{
    constexpr int KP = 8 * SPT;
    extern __shared__ float2 sm2[];
    float2 *Xs = sm2;                  // [KP][kXS]
    float2 *Vs = Xs + KP * kXS;        // [kb][kVS]
    float2 *Bs = Vs;                   // [kTileC][kBS]   (after backward)
    float2 *Rs = Vs;                   // [32][KP]        (after forward)

    hs_pdl_launch_next();
    const int pat = blockIdx.y;
    const int tile = a.f.chunk_base + blockIdx.x;
    const int tid = threadIdx.x;
    const int kb = hs_tile_kb(a.n);
    const int packed = __ldg(a.tiles + tile);
    const int r0 = packed >> 16, c0 = packed & 0xffff;
    const float2 *gx = a.gx + (int64_t)pat * a.tab_stride;
    const float2 *gy = a.gy + (int64_t)pat * a.tab_stride;
    const float2 *cf = a.coef + (int64_t)pat * a.np;

    // ---- stage X[k][c] (k < KP) and V[k][r] = coef_k gy[r][k] (k < kb).
    // Warp w takes columns / rows w + 8 i; lane l spots l + 32 m.  All of a
    // thread's global loads are issued before its shared stores (deep MLP).
    {
        constexpr int MK = (KP + 31) / 32;
        const int lane = tid & 31, warp = tid >> 5;
        float2 v[8][MK];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 *src = gx + (int64_t)min(c0 + warp + 8 * i, a.side - 1) * a.np;
#pragma unroll
            for (int m = 0; m < MK; ++m) {
                const int k = lane + 32 * m;
                v[i][m] = (k < KP) ? __ldg(src + k) : make_float2(0.f, 0.f);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int m = 0; m < MK; ++m) {
                const int k = lane + 32 * m;
                if (k < KP) Xs[k * kXS + warp + 8 * i] = v[i][m];
            }
        // -- below: the previous pass's results (status, coef)
        hs_pdl_wait_prev();
        if (a.f.u.status[pat] != 0) return;  // uniform per CTA
        float2 w[MK];
#pragma unroll
        for (int m = 0; m < MK; ++m) {
            const int k = lane + 32 * m;
            w[m] = (k < kb) ? __ldg(cf + k) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 *src = gy + (int64_t)min(r0 + warp + 8 * i, a.side - 1) * a.np;
#pragma unroll
            for (int m = 0; m < MK; ++m) {
                const int k = lane + 32 * m;
                v[i][m] = (k < kb) ? __ldg(src + k) : make_float2(0.f, 0.f);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int m = 0; m < MK; ++m) {
                const int k = lane + 32 * m;
                const float2 q = v[i][m];
                if (k < kb)
                    Vs[k * kVS + warp + 8 * i] =
                        make_float2(fmaf(w[m].x, q.x, -w[m].y * q.y), fmaf(w[m].x, q.y, w[m].y * q.x));
            }
    }
    __syncthreads();

    // ---- backward: thread (tr, tc) holds rows 4 tr + i, columns tc + 16 j
    const int tr = tid >> 4, tc = tid & 15;
    f2x sacc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sacc[i][j] = 0ull;
    const f2x *X2 = reinterpret_cast<const f2x *>(Xs);
#pragma unroll 16
    for (int k = 0; k < kb; ++k) {
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

    // ---- b = A conj(S)/|S| (arg(0) = 0); optional phase write
    float br[4][4], bi[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = r0 + 4 * tr + i, c = c0 + tc + 16 * j;
            const bool in = (r < a.side) && (c < a.side);
            const int64_t gidx = (int64_t)r * a.side + c;
            const float A = in ? __ldg(a.amp_img + gidx) : 0.f;
            const float x = f2_lo(sacc[i][j]), y = f2_hi(sacc[i][j]);
            hs_bvec_exact(x, y, A, br[i][j], bi[i][j]);
            if (WRITE && in) {
                const int32_t di = __ldg(a.idx_img + gidx);
                if (di >= 0) {
                    hs_store_phase(a.phase_out, a.phase_out32, (int64_t)pat * a.phase_stride + di, x, y);
                    if (a.raster)
                        a.raster[(int64_t)pat * a.side * a.side + gidx] = hs_gray_linear(hs_phase_f64(x, y));
                }
            }
        }
    __syncthreads();  // V no longer read: its space becomes b [c][r]
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float4 *dst = reinterpret_cast<float4 *>(Bs + (tc + 16 * j) * kBS + 4 * tr);
        dst[0] = make_float4(br[0][j], bi[0][j], br[1][j], bi[1][j]);
        dst[1] = make_float4(br[2][j], bi[2][j], br[3][j], bi[3][j]);
    }
    __syncthreads();

    // ---- forward: thread (rg, sg) holds rows 2 rg, 2 rg + 1 x spots sg + 8 j
    const int rg = tid >> 3, sg = tid & 7;
    f2x t0[SPT], t1[SPT];
#pragma unroll
    for (int j = 0; j < SPT; ++j) t0[j] = t1[j] = 0ull;
#pragma unroll 16
    for (int c = 0; c < kTileC; ++c) {
        const float4 b = *reinterpret_cast<const float4 *>(Bs + c * kBS + 2 * rg);
        f2x x[SPT];
#pragma unroll
        for (int j = 0; j < SPT; ++j) x[j] = X2[(sg + 8 * j) * kXS + c];
#pragma unroll
        for (int j = 0; j < SPT; ++j) f2_cmac(t0[j], b.x, b.y, x[j]);
#pragma unroll
        for (int j = 0; j < SPT; ++j) f2_cmac(t1[j], b.z, b.w, x[j]);
    }
    // E_k = sum_i gy[r][k] T[i][k] over the thread's two rows
    const int ra = min(r0 + 2 * rg, a.side - 1), rb = min(r0 + 2 * rg + 1, a.side - 1);
    f2x e2[SPT];
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
        const int k = sg + 8 * j;
        const float2 qa = __ldg(gy + (int64_t)ra * a.np + k);
        const float2 qb = __ldg(gy + (int64_t)rb * a.np + k);
        e2[j] = 0ull;
        f2_cmac(e2[j], qa.x, qa.y, t0[j]);
        f2_cmac(e2[j], qb.x, qb.y, t1[j]);
    }
    __syncthreads();  // b no longer read: its space becomes the row-group partials
#pragma unroll
    for (int j = 0; j < SPT; ++j) reinterpret_cast<f2x *>(Rs)[rg * KP + sg + 8 * j] = e2[j];
    __syncthreads();
    float2 *out = a.f.partials + (int64_t)pat * a.f.part_stride + (int64_t)tile * a.np;
    for (int k = tid; k < a.np; k += kThreads) {
        float x = 0.f, y = 0.f;
        if (k < KP) {
#pragma unroll 16
            for (int q = 0; q < 32; ++q) {
                const float2 v = Rs[q * KP + k];
                x += v.x;
                y += v.y;
            }
        }
        out[k] = make_float2(x, y);
    }
    if (a.f.u.act != ACT_NONE) {
        __syncthreads();
        hs_fold(a.f, pat, tile, reinterpret_cast<char *>(Vs));
    }
}

typedef void (*TileFn)(TileArgs);
TileFn hs_select_tile(int spt, bool write);

}  // namespace hs
