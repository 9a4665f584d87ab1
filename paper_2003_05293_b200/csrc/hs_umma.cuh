// hs_umma.cuh -- full-range fused pass on the tcgen05 tensor cores.
//
// Same pass as hs_tile.cuh (backward kernels.py:99-119, b = A conj(S)/|S|
// kernels.py:136-137, forward kernels.py:122-144) for np <= 112, with both
// complex GEMMs of a 128-row x 64-column tile issued as tcgen05.mma
// kind::tf32 (M = 128) and accumulated in TMEM:
//
//   backward  S[r][c] = sum_k gy[r0+r][k] X'[c][k]   gy planes (A, smem, TMA)
//                                                    X' = coef_k gx[c0+c][k] (B, smem)
//   b         = A conj(S)/|S| (registers), phase write
//   forward   T[r][k] = sum_c b[r][c] X[c][k]   b (A, smem), X^T (B, smem)
//   E_k       = sum_r gy[r0+r][k] T[r][k]       (CUDA cores, fixed-order reduce)
//
// FP32 accuracy from TF32 units: every operand is split x = hi + lo with
// hi = rna_tf32(x), and each real product is hi*hi + hi*lo + lo*hi (the
// dropped lo*lo term is ~2^-22 relative).  A complex MAC is four real
// products (Sr = Vr Xr - Vi Xi: the minus via the instruction's a_negate
// bit), so one 8-deep k-step is 12 MMAs per accumulator pair.
//
// Two CTAs per SM (256 TMEM columns each), so one CTA's CUDA-core phases
// (operand builds, b, the E reduce, the fold) overlap the other's MMAs:
//   TMEM [0, 128)     S = {Sr, Si} x 64 columns                            backward
//        [0, 2 NP)    T = {Tr, Ti} x NP spots                              forward
// S is read once into registers (b: 32 columns per thread), which frees the
// columns T reuses.  The backward's A operand gy is constant for the whole
// solve: hs_umma_prep_kernel writes its tf32 hi/lo planes once per table
// build, already in the shared-memory operand layout, and each k-step's
// 16 KB block is one TMA bulk copy (issued one chunk ahead); the per-pass
// coefficients go on the B side (coef_k gx[c][k], built by the threads).
// The same planes give the E epilogue coalesced gy reads (hi + lo == gy
// exactly).  Shared memory: a ring of three operand stages, each either a
// backward k-step (gy: 128 rows x 8 spots, X: 64 columns x 8 spots) or a
// forward k-step (b': 128 rows x 8 columns, X^T: NP spots x 8 columns), 4
// planes each, in the SWIZZLE_NONE K-major canonical layout (8 x 16-byte
// core matrices).  One thread issues the MMAs and commits each stage to its
// mbarrier; the threads wait for the MMAs two stages back before reusing a
// stage, so the tensor pipe always has the previous k-step queued.
//
// Encodings (instruction descriptor, shared-memory descriptor, TMEM
// st / ld, a_negate) are checked by tools/umma_probe.cu.
#pragma once

#include "hs_kernels.cuh"
#include "hs_tile.cuh"

namespace hs {

constexpr int kUR = 128;         // tile rows (MMA M)
constexpr int kUC = 64;          // tile columns
constexpr int kUF = 8;           // spots / columns per stage (one MMA k-step)
constexpr int kUNPMax = 112;     // largest np (TMEM: 2 np <= 256)
constexpr int kUThreads = 256;
constexpr int kUTmem = 256;      // TMEM columns per CTA (two CTAs per SM)
constexpr int kUStages = 3;
constexpr int kUAPl = kUR * kUF * 4;                // A plane [128][8] (4 KB)
constexpr int kUBOff = 4 * kUAPl;                   // B planes after the 4 A planes
constexpr int kUSlot = kUBOff + 4 * kUNPMax * kUF * 4;  // 30 KB: b' + X^T at np = 112
constexpr int kUPlaneBlock = 4 * kUAPl;             // gy planes of one (band, k-step): 16 KB

__host__ __device__ constexpr size_t hs_umma_smem_bytes()
{
    // operand stages + 1 KB alignment + E reduce scratch [8 warps][64] float
    return kUStages * (size_t)kUSlot + 1024 + 8 * 64 * sizeof(float);
}

// gy planes of one pattern: [band][k-step][4][128 rows][8 spots] floats
__host__ __device__ constexpr int64_t hs_umma_plane_floats(int side, int np)
{
    return (int64_t)((side + kUR - 1) / kUR) * (np / kUF) * (kUPlaneBlock / 4);
}

// Offset (floats) of element (r, k) in a [128][8] K-major operand plane.
__host__ __device__ constexpr int hs_uoff(int r, int k) { return r * 4 + (k >> 2) * 512 + (k & 3); }

// gy -> tf32 hi/lo planes {re_h, re_l, im_h, im_l} in the operand layout.
// grid (bands * np / 8, B), 256 threads.
static __global__ void hs_umma_prep_kernel(const float2 *__restrict__ gy, float *__restrict__ planes, int side,
                                           int np, int64_t tab_stride, int64_t plane_stride)
{
    const int nks = np / kUF;
    const int band = blockIdx.x / nks, ks = blockIdx.x % nks;
    const int pat = blockIdx.y;
    float *dst = planes + (int64_t)pat * plane_stride + (int64_t)blockIdx.x * (kUPlaneBlock / 4);
    for (int i = threadIdx.x; i < kUR * kUF; i += blockDim.x) {
        const int r = i / kUF, k = i % kUF;
        const int grow = band * kUR + r;
        float2 v = make_float2(0.f, 0.f);
        if (grow < side) v = gy[(int64_t)pat * tab_stride + (int64_t)grow * np + ks * kUF + k];
        uint32_t hr, hi;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hr) : "f"(v.x));
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(v.y));
        const int o = hs_uoff(r, k);
        dst[o] = __uint_as_float(hr);
        dst[o + kUAPl / 4] = v.x - __uint_as_float(hr);
        dst[o + 2 * kUAPl / 4] = __uint_as_float(hi);
        dst[o + 3 * kUAPl / 4] = v.y - __uint_as_float(hi);
    }
}

// ---- PTX wrappers --------------------------------------------------------
__device__ __forceinline__ uint64_t hs_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);  // sm100 version, no swizzle
}

// kind::tf32, f32 accumulate, A and B K-major
__host__ __device__ constexpr uint32_t hs_idesc_tf32(int n, bool neg)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((neg ? 1u : 0u) << 13) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(kUR >> 4) << 24);
}

// A from TMEM
__device__ __forceinline__ void hs_mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

// A from shared memory
__device__ __forceinline__ void hs_mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void hs_tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void hs_tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void hs_tc_st8(uint32_t taddr, const float (&v)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

__device__ __forceinline__ void hs_tc_ld8(uint32_t taddr, float (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(taddr)
                 : "memory");
}

__device__ __forceinline__ void hs_tc_ld4(uint32_t taddr, float *v)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                 : "r"(taddr)
                 : "memory");
}

__device__ __forceinline__ void hs_tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void hs_tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float hs_tf32_hi(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// hi/lo split of 4 values into two float4
__device__ __forceinline__ void hs_split4(float a, float b, float c, float d, float4 &hi, float4 &lo)
{
    hi = make_float4(hs_tf32_hi(a), hs_tf32_hi(b), hs_tf32_hi(c), hs_tf32_hi(d));
    lo = make_float4(a - hi.x, b - hi.y, c - hi.z, d - hi.w);
}

__device__ __forceinline__ void hs_mbar_wait(uint32_t bar, uint32_t parity)
{
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(bar), "r"(parity)
                     : "memory");
}

// Issue the 12 real MMAs of one complex k-step:
//   Dr += Ar Br - Ai Bi,  Di += Ar Bi + Ai Br   (each as hi*hi + hi*lo + lo*hi)
// A planes {Ar_h, Ar_l, Ai_h, Ai_l} given by `aop(p)` (TMEM address or smem
// descriptor), B planes {Br_h, Br_l, Bi_h, Bi_l} as smem descriptors.
template <typename AOp, typename Mma>
__device__ __forceinline__ void hs_cmma(Mma mma, uint32_t dr, uint32_t di, AOp aop, const uint64_t (&b)[4],
                                        uint32_t id, uint32_t idn, uint32_t acc)
{
    mma(dr, aop(0), b[0], id, acc);
    mma(dr, aop(0), b[1], id, 1u);
    mma(dr, aop(1), b[0], id, 1u);
    mma(dr, aop(2), b[2], idn, 1u);
    mma(dr, aop(2), b[3], idn, 1u);
    mma(dr, aop(3), b[2], idn, 1u);
    mma(di, aop(0), b[2], id, acc);
    mma(di, aop(0), b[3], id, 1u);
    mma(di, aop(1), b[2], id, 1u);
    mma(di, aop(2), b[0], id, 1u);
    mma(di, aop(2), b[1], id, 1u);
    mma(di, aop(3), b[0], id, 1u);
}

template <int NP, bool WRITE>
__global__ void __launch_bounds__(kUThreads, 2) hs_umma_kernel(const TileArgs a)
{
    static_assert(NP % 16 == 0 && NP <= kUNPMax, "forward N = np must be a multiple of 16, <= 112");
    constexpr int NCC = kUC / kUF;           // forward k-steps (8)
    constexpr uint32_t BPL = kUC * kUF * 4;  // backward X plane bytes (2 KB)
    constexpr uint32_t FPL = NP * kUF * 4;   // forward X^T plane bytes
    constexpr uint32_t FLBO = (NP / 8) * 128;
    constexpr int KH = NP / 2;               // spots per thread in the E epilogue
    extern __shared__ __align__(1024) unsigned char smu[];
    __shared__ __align__(8) unsigned long long mbar[2 * kUStages];  // [0, 3) MMA done, [3, 6) TMA full
    __shared__ uint32_t s_tmem;
    __shared__ float2 coef_s[NP];

    hs_pdl_launch_next();
    const int pat = blockIdx.y;
    const int tile = a.f.chunk_base + blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = warp & 3, h = warp >> 2;  // TMEM lane quarter, column / spot half
    const int row = 32 * q + lane;          // tile row of this thread (TMEM lane)
    const int packed = __ldg(a.tiles + tile);
    const int r0 = packed >> 16, c0 = packed & 0xffff;
    const float2 *gx = a.gx + (int64_t)pat * a.tab_stride;
    const float *gyp = a.gyp + (int64_t)pat * a.gyp_stride + (int64_t)(r0 / kUR) * (NP / kUF) * (kUPlaneBlock / 4);
    const int n = a.n;
    const int ksteps = (n + 7) / 8;          // backward k-steps (8 spots)
    const int nsteps = ksteps + NCC;         // stage sequence: backward, then forward

    unsigned char *sbase = reinterpret_cast<unsigned char *>(((uintptr_t)smu + 1023) & ~(uintptr_t)1023);
    const uint32_t sb = hs_smem_addr(sbase);
    float *red = reinterpret_cast<float *>(sbase + kUStages * kUSlot);  // [8][64]
    const int grow = r0 + row;
    const bool row_in = grow < a.side;

    // ---- backward X loads: thread (column c = tid / 2, spot quad kq = tid % 2)
    // of threads < 128 loads spots 8 ks + 4 kq .. + 4 of gx[c0 + c]
    const bool xb_on = tid < 2 * kUC;
    const int xb_c = (tid >> 1) & (kUC - 1), xb_kq = tid & 1;
    const float4 *xb_src = reinterpret_cast<const float4 *>(gx + (int64_t)min(c0 + xb_c, a.side - 1) * a.np);
    float4 xb0 = make_float4(0.f, 0.f, 0.f, 0.f), xb1 = xb0;
    auto load_b = [&](int ks) {
        const int k = ks * kUF + 4 * xb_kq;
        if (xb_on) {
            xb0 = __ldg(xb_src + k / 2);
            xb1 = __ldg(xb_src + k / 2 + 1);
        }
    };
    load_b(0);  // gx: an input of the whole solve

    // -- below: the previous pass's results (status, coef); TMEM is taken
    // only now, so a dependent-launched CTA never holds it while waiting
    hs_pdl_wait_prev();
    if (a.f.u.status[pat] != 0) return;  // uniform per CTA
    if (tid < NP) coef_s[tid] = (tid < n) ? a.coef[(int64_t)pat * a.np + tid] : make_float2(0.f, 0.f);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(hs_smem_addr(&s_tmem)),
                     "n"(kUTmem));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const uint32_t bar = hs_smem_addr(&mbar[0]);  // stage s: MMA done bar + 8 s, TMA full bar + 8 (3 + s)
    auto tma_gy = [&](int ks) {  // gy planes of k-step ks -> stage ks % 3 (thread 0)
        const int s = ks % kUStages;
        const uint32_t fb = bar + 8 * (kUStages + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "n"(kUPlaneBlock) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sb + s * kUSlot),
                     "l"(gyp + (int64_t)ks * (kUPlaneBlock / 4)), "n"(kUPlaneBlock), "r"(fb)
                     : "memory");
    };
    if (tid == 0) {
        for (int i = 0; i < 2 * kUStages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8 * i));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma_gy(0);
    }
    hs_tc_fence_before();
    __syncthreads();
    hs_tc_fence_after();
    const uint32_t tm = s_tmem;
    const uint32_t tl = tm + ((uint32_t)(32 * q) << 16);  // this warp's lane quarter

    // MMA completion of stage-sequence step j is completion (j / 3) of
    // barrier j % 3; waits happen in order, never two phases behind.
    int done = 0;  // steps known complete
    auto wait_mma = [&](int j) {
        for (; done <= j; ++done) hs_mbar_wait(bar + 8 * (done % kUStages), (uint32_t)(done / kUStages) & 1u);
        hs_tc_fence_after();
    };
    auto commit = [&](int j) {  // thread 0, after issuing step j's MMAs
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         bar + 8 * (j % kUStages))
                     : "memory");
    };
    // operands written by the threads (generic proxy) become visible to the
    // MMA-issuing thread (async proxy)
    auto publish = [&]() {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        hs_tc_fence_before();
        __syncthreads();
        hs_tc_fence_after();
    };
    auto mma_ss = [](uint32_t d, uint64_t av, uint64_t bv, uint32_t id, uint32_t acc) { hs_mma_ss(d, av, bv, id, acc); };

    // ---- backward: S = gy (coef X)^T ------------------------------------------
    const uint32_t idb = hs_idesc_tf32(kUC, false), idbn = hs_idesc_tf32(kUC, true);
    for (int ks = 0; ks < ksteps; ++ks) {
        const int s = ks % kUStages;
        if (ks >= 2) wait_mma(ks - 2);  // stage of ks + 1 (and of ks) free
        if (tid == 0 && ks + 1 < ksteps) tma_gy(ks + 1);
        if (xb_on) {  // X' = coef_k gx[c][k], planes [64 columns][8 spots]: (c/8)*128 + (k/4)*1024 + (c%8)*16
            const int k = ks * kUF + 4 * xb_kq;
            const float2 w0 = coef_s[k], w1 = coef_s[k + 1], w2 = coef_s[k + 2], w3 = coef_s[k + 3];
            const float xr0 = fmaf(w0.x, xb0.x, -w0.y * xb0.y), xi0 = fmaf(w0.x, xb0.y, w0.y * xb0.x);
            const float xr1 = fmaf(w1.x, xb0.z, -w1.y * xb0.w), xi1 = fmaf(w1.x, xb0.w, w1.y * xb0.z);
            const float xr2 = fmaf(w2.x, xb1.x, -w2.y * xb1.y), xi2 = fmaf(w2.x, xb1.y, w2.y * xb1.x);
            const float xr3 = fmaf(w3.x, xb1.z, -w3.y * xb1.w), xi3 = fmaf(w3.x, xb1.w, w3.y * xb1.z);
            float4 rh, rl, ih, il;
            hs_split4(xr0, xr1, xr2, xr3, rh, rl);
            hs_split4(xi0, xi1, xi2, xi3, ih, il);
            unsigned char *d = sbase + s * kUSlot + kUBOff + (xb_c >> 3) * 128 + xb_kq * 1024 + (xb_c & 7) * 16;
            *reinterpret_cast<float4 *>(d) = rh;
            *reinterpret_cast<float4 *>(d + BPL) = rl;
            *reinterpret_cast<float4 *>(d + 2 * BPL) = ih;
            *reinterpret_cast<float4 *>(d + 3 * BPL) = il;
        }
        if (ks + 1 < ksteps) load_b(ks + 1);  // next k-step's loads in flight across the publish
        publish();
        if (tid == 0) {
            hs_mbar_wait(bar + 8 * (kUStages + s), (uint32_t)(ks / kUStages) & 1u);  // gy planes landed
            const uint32_t xs = sb + s * kUSlot;
            const uint64_t xb[4] = {hs_sdesc(xs + kUBOff, 1024, 128), hs_sdesc(xs + kUBOff + BPL, 1024, 128),
                                    hs_sdesc(xs + kUBOff + 2 * BPL, 1024, 128),
                                    hs_sdesc(xs + kUBOff + 3 * BPL, 1024, 128)};
            hs_cmma(mma_ss, tm, tm + kUC, [&](int pl) { return hs_sdesc(xs + pl * kUAPl, 2048, 128); }, xb, idb,
                    idbn, ks ? 1u : 0u);
            commit(ks);
        }
    }

    // ---- forward X^T loads: item (spot k = tid / 2, column quad cq = tid % 2):
    // gx[c0 + 8 cc + 4 cq + j][k], j < 4 ---------------------------------------
    const int xf_k = tid >> 1, xf_cq = tid & 1;
    const bool xf_on = xf_k < NP;
    float2 xf[4];
    auto load_f = [&](int cc) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gc = min(c0 + cc * kUF + 4 * xf_cq + j, a.side - 1);
            xf[j] = (xf_on && xf_k < n) ? __ldg(gx + (int64_t)gc * a.np + xf_k) : make_float2(0.f, 0.f);
        }
    };
    load_f(0);

    // amplitudes of this thread's 32 pixels: columns 8 cc + 4 h + j (c0 is a
    // multiple of 4, so each group of 4 is one aligned float4 when side % 4 == 0)
    const int64_t prow = (int64_t)min(grow, a.side - 1) * a.side;
    float br[32], bi[32];
    const bool vec_amp = (a.side & 3) == 0;
#pragma unroll
    for (int cc = 0; cc < NCC; ++cc) {
        const int c = c0 + cc * kUF + 4 * h;
        if (vec_amp) {
            const float4 v = (row_in && c < a.side) ? __ldg(reinterpret_cast<const float4 *>(a.amp_img + prow + c))
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            br[4 * cc] = v.x; br[4 * cc + 1] = v.y; br[4 * cc + 2] = v.z; br[4 * cc + 3] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                br[4 * cc + j] = (row_in && c + j < a.side) ? __ldg(a.amp_img + prow + c + j) : 0.f;
        }
    }
    wait_mma(ksteps - 1);

    // ---- S -> b = A conj(S)/|S| (registers), phase write --------------------
#pragma unroll
    for (int cc = 0; cc < NCC; cc += 2) {
        float sr[8], si[8];
        hs_tc_ld4(tl + cc * kUF + 4 * h, sr);
        hs_tc_ld4(tl + (cc + 1) * kUF + 4 * h, sr + 4);
        hs_tc_ld4(tl + kUC + cc * kUF + 4 * h, si);
        hs_tc_ld4(tl + kUC + (cc + 1) * kUF + 4 * h, si + 4);
        hs_tc_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int i = 4 * cc + jj;
            const float A = br[i];
            hs_bvec_exact(sr[jj], si[jj], A, br[i], bi[i]);
            if (WRITE) {
                const int c = c0 + (i / 4) * kUF + 4 * h + (i % 4);
                if (row_in && c < a.side) {
                    const int32_t di = __ldg(a.idx_img + prow + c);
                    if (di >= 0) {
                        const double ph = hs_phase_f64(sr[jj], si[jj]);
                        a.phase_out[(int64_t)pat * a.phase_stride + di] = ph;
                        if (a.raster) a.raster[(int64_t)pat * a.side * a.side + prow + c] = hs_gray_linear(ph);
                    }
                }
            }
        }
    }

    // ---- forward: T = b X ------------------------------------------------------
    // stage: b' planes [128 rows][8 columns] (hs_uoff), then X^T planes
    // [NP spots][8 columns] ((k/8)*128 + (c/4)*FLBO + (k%8)*16 + (c%4)*4)
    const uint32_t idf = hs_idesc_tf32(NP, false), idfn = hs_idesc_tf32(NP, true);
#pragma unroll
    for (int cc = 0; cc < NCC; ++cc) {
        const int j = ksteps + cc;  // stage-sequence step
        const int s = j % kUStages;
        if (j >= 3) wait_mma(j - 3);  // this stage free
        unsigned char *slot = sbase + s * kUSlot;
        {   // b' (this thread's row, columns 4h .. 4h+3 of the k-step)
            float4 rh, rl, ih, il;
            hs_split4(br[4 * cc], br[4 * cc + 1], br[4 * cc + 2], br[4 * cc + 3], rh, rl);
            hs_split4(bi[4 * cc], bi[4 * cc + 1], bi[4 * cc + 2], bi[4 * cc + 3], ih, il);
            unsigned char *d = slot + row * 16 + h * 2048;
            *reinterpret_cast<float4 *>(d) = rh;
            *reinterpret_cast<float4 *>(d + kUAPl) = rl;
            *reinterpret_cast<float4 *>(d + 2 * kUAPl) = ih;
            *reinterpret_cast<float4 *>(d + 3 * kUAPl) = il;
        }
        if (xf_on) {
            float4 rh, rl, ih, il;
            hs_split4(xf[0].x, xf[1].x, xf[2].x, xf[3].x, rh, rl);
            hs_split4(xf[0].y, xf[1].y, xf[2].y, xf[3].y, ih, il);
            unsigned char *d = slot + kUBOff + (xf_k >> 3) * 128 + xf_cq * FLBO + (xf_k & 7) * 16;
            *reinterpret_cast<float4 *>(d) = rh;
            *reinterpret_cast<float4 *>(d + FPL) = rl;
            *reinterpret_cast<float4 *>(d + 2 * FPL) = ih;
            *reinterpret_cast<float4 *>(d + 3 * FPL) = il;
        }
        if (cc + 1 < NCC) load_f(cc + 1);
        publish();  // (cc = 0: also orders the S reads before T overwrites S)
        if (tid == 0) {
            const uint32_t xs = sb + s * kUSlot;
            const uint64_t xb[4] = {hs_sdesc(xs + kUBOff, FLBO, 128), hs_sdesc(xs + kUBOff + FPL, FLBO, 128),
                                    hs_sdesc(xs + kUBOff + 2 * FPL, FLBO, 128),
                                    hs_sdesc(xs + kUBOff + 3 * FPL, FLBO, 128)};
            hs_cmma(mma_ss, tm, tm + NP, [&](int pl) { return hs_sdesc(xs + pl * kUAPl, 2048, 128); }, xb, idf,
                    idfn, cc ? 1u : 0u);
            commit(j);
        }
    }
    wait_mma(nsteps - 1);

    // ---- E_k = sum_r gy[r][k] T[r][k]: spots KH h .. KH (h+1) of the row in
    // two 8-aligned parts (KA + KB = KH, KA <= 32); each part is
    // transpose-reduced over the warp's 32 rows (64 padded values -> 2 per
    // lane), then the 4 lane-quarter warps are summed in order through shared
    // memory.  gy comes from the planes (hi + lo), coalesced over the rows.
    float2 *out = a.f.partials + (int64_t)pat * a.f.part_stride + (int64_t)tile * a.np;
    constexpr int KA = 8 * ((KH / 8 + 1) / 2), KB = KH - KA;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
        const int KQ = part ? KB : KA;
        if (KQ == 0) break;  // compile-time per NP
        const int kbase = KH * h + (part ? KA : 0);
        float v[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) v[j] = 0.f;
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
            if (8 * k8 < KQ) {
                const int kk = kbase + 8 * k8;  // multiple of 8: one plane block
                const float4 *pb = reinterpret_cast<const float4 *>(gyp + (int64_t)(kk / kUF) * (kUPlaneBlock / 4)) + row;
                float gr[8], gi[8];
#pragma unroll
                for (int hq = 0; hq < 2; ++hq) {  // spots 4 hq .. 4 hq + 3 at float4 offset hq * 128
                    const float4 rh = __ldg(pb + hq * 128), rl = __ldg(pb + 256 + hq * 128);
                    const float4 ih = __ldg(pb + 512 + hq * 128), il = __ldg(pb + 768 + hq * 128);
                    gr[4 * hq] = rh.x + rl.x; gr[4 * hq + 1] = rh.y + rl.y;
                    gr[4 * hq + 2] = rh.z + rl.z; gr[4 * hq + 3] = rh.w + rl.w;
                    gi[4 * hq] = ih.x + il.x; gi[4 * hq + 1] = ih.y + il.y;
                    gi[4 * hq + 2] = ih.z + il.z; gi[4 * hq + 3] = ih.w + il.w;
                }
                float tr[8], ti[8];
                hs_tc_ld8(tl + kk, tr);
                hs_tc_ld8(tl + NP + kk, ti);
                hs_tc_wait_ld();
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    v[16 * k8 + 2 * j] = fmaf(gr[j], tr[j], -gi[j] * ti[j]);
                    v[16 * k8 + 2 * j + 1] = fmaf(gr[j], ti[j], gi[j] * tr[j]);
                }
            }
        }
        // transpose-reduce: at offset o the lane keeps the half selected by
        // its lane bit o (a fixed order per value: deterministic)
#pragma unroll
        for (int o = 16, w = 32; o > 0; o >>= 1, w >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int j = 0; j < w; ++j) {
                const float send = up ? v[j] : v[j + w];
                const float keep = up ? v[j + w] : v[j];
                v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        const int base = ((lane & 16) ? 32 : 0) + ((lane & 8) ? 16 : 0) + ((lane & 4) ? 8 : 0) +
                         ((lane & 2) ? 4 : 0) + ((lane & 1) ? 2 : 0);
        red[warp * 64 + base] = v[0];
        red[warp * 64 + base + 1] = v[1];
        __syncthreads();
        // value 2 j (+1) of part (hq, part) is spot KH hq + kbase-offset + j
        if (tid < 2 * 32) {
            const int hq = tid >> 5, j = tid & 31;
            if (j < KQ) {
                float x = 0.f, y = 0.f;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    x += red[(qq + 4 * hq) * 64 + 2 * j];
                    y += red[(qq + 4 * hq) * 64 + 2 * j + 1];
                }
                out[KH * hq + (part ? KA : 0) + j] = make_float2(x, y);
            }
        }
        __syncthreads();
    }

    hs_tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(kUTmem));
    if (a.f.u.act != ACT_NONE) hs_fold(a.f, pat, tile, reinterpret_cast<char *>(sbase));
}

typedef void (*UmmaFn)(TileArgs);
UmmaFn hs_select_umma(int np, bool write);

}  // namespace hs
