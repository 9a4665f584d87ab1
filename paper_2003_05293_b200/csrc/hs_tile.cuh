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
    const float2 *coef;       // [B][np]
    const float *amp_img;     // [side][side], 0 outside the aperture
    const int32_t *idx_img;   // [side][side] storage index, -1 outside
    double *phase_out;        // [B][phase_stride] (WRITE)
    unsigned char *raster;    // [B][side][side] SLM gray raster (WRITE, nullable)
    int64_t phase_stride;
    FoldArgs f;
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

    const int pat = blockIdx.y;
    const int tile = a.f.chunk_base + blockIdx.x;
    if (a.f.u.status[pat] != 0) return;
    const int tid = threadIdx.x;
    const int kb = hs_tile_kb(a.n);
    const int packed = __ldg(a.tiles + tile);
    const int r0 = packed >> 16, c0 = packed & 0xffff;
    const float2 *gx = a.gx + (int64_t)pat * a.tab_stride;
    const float2 *gy = a.gy + (int64_t)pat * a.tab_stride;
    const float2 *cf = a.coef + (int64_t)pat * a.np;

    // ---- stage X[k][c] (k < KP) and V[k][r] = coef_k gy[r][k] (k < kb); reads coalesced over k
    for (int idx = tid; idx < KP * kTileC; idx += kThreads) {
        const int c = idx / KP, k = idx - c * KP;
        const int cc = min(c0 + c, a.side - 1);
        Xs[k * kXS + c] = __ldg(gx + (int64_t)cc * a.np + k);
    }
    for (int idx = tid; idx < kb * kTileR; idx += kThreads) {
        const int r = idx / kb, k = idx - r * kb;
        const int rr = min(r0 + r, a.side - 1);
        const float2 q = __ldg(gy + (int64_t)rr * a.np + k);
        const float2 w = __ldg(cf + k);
        Vs[k * kVS + r] = make_float2(fmaf(w.x, q.x, -w.y * q.y), fmaf(w.x, q.y, w.y * q.x));
    }
    __syncthreads();

    // ---- backward: thread (tr, tc) holds rows 4 tr + i, columns tc + 16 j
    const int tr = tid >> 4, tc = tid & 15;
    float sr[4][4], si[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sr[i][j] = si[i][j] = 0.f;
#pragma unroll 2
    for (int k = 0; k < kb; ++k) {
        const float4 v01 = *reinterpret_cast<const float4 *>(Vs + k * kVS + 4 * tr);
        const float4 v23 = *reinterpret_cast<const float4 *>(Vs + k * kVS + 4 * tr + 2);
        float2 x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = Xs[k * kXS + tc + 16 * j];
        const float vr[4] = {v01.x, v01.z, v23.x, v23.z};
        const float vi[4] = {v01.y, v01.w, v23.y, v23.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                sr[i][j] = fmaf(vr[i], x[j].x, sr[i][j]);
                si[i][j] = fmaf(vr[i], x[j].y, si[i][j]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                sr[i][j] = fmaf(-vi[i], x[j].y, sr[i][j]);
                si[i][j] = fmaf(vi[i], x[j].x, si[i][j]);
            }
        }
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
            const float x = sr[i][j], y = si[i][j];
            hs_bvec_exact(x, y, A, br[i][j], bi[i][j]);
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
    float tr0[SPT], ti0[SPT], tr1[SPT], ti1[SPT];
#pragma unroll
    for (int j = 0; j < SPT; ++j) tr0[j] = ti0[j] = tr1[j] = ti1[j] = 0.f;
#pragma unroll 2
    for (int c = 0; c < kTileC; ++c) {
        const float4 b = *reinterpret_cast<const float4 *>(Bs + c * kBS + 2 * rg);
        float2 x[SPT];
#pragma unroll
        for (int j = 0; j < SPT; ++j) x[j] = Xs[(sg + 8 * j) * kXS + c];
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            tr0[j] = fmaf(b.x, x[j].x, tr0[j]);
            ti0[j] = fmaf(b.x, x[j].y, ti0[j]);
        }
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            tr0[j] = fmaf(-b.y, x[j].y, tr0[j]);
            ti0[j] = fmaf(b.y, x[j].x, ti0[j]);
        }
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            tr1[j] = fmaf(b.z, x[j].x, tr1[j]);
            ti1[j] = fmaf(b.z, x[j].y, ti1[j]);
        }
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            tr1[j] = fmaf(-b.w, x[j].y, tr1[j]);
            ti1[j] = fmaf(b.w, x[j].x, ti1[j]);
        }
    }
    // E_k = sum_i gy[r][k] T[i][k] over the thread's two rows
    const int ra = min(r0 + 2 * rg, a.side - 1), rb = min(r0 + 2 * rg + 1, a.side - 1);
    float er[SPT], ei[SPT];
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
        const int k = sg + 8 * j;
        const float2 qa = __ldg(gy + (int64_t)ra * a.np + k);
        const float2 qb = __ldg(gy + (int64_t)rb * a.np + k);
        float x = qa.x * tr0[j];
        x = fmaf(-qa.y, ti0[j], x);
        x = fmaf(qb.x, tr1[j], x);
        x = fmaf(-qb.y, ti1[j], x);
        float y = qa.x * ti0[j];
        y = fmaf(qa.y, tr0[j], y);
        y = fmaf(qb.x, ti1[j], y);
        y = fmaf(qb.y, tr1[j], y);
        er[j] = x;
        ei[j] = y;
    }
    __syncthreads();  // b no longer read: its space becomes the row-group partials
#pragma unroll
    for (int j = 0; j < SPT; ++j) Rs[rg * KP + sg + 8 * j] = make_float2(er[j], ei[j]);
    __syncthreads();
    float2 *out = a.f.partials + (int64_t)pat * a.f.part_stride + (int64_t)tile * a.np;
    for (int k = tid; k < a.np; k += kThreads) {
        float x = 0.f, y = 0.f;
        if (k < KP) {
#pragma unroll 8
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
