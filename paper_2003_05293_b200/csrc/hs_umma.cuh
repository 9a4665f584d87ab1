// hs_umma.cuh -- full-range fused pass on the tcgen05 tensor cores.
//
// Same pass as hs_tile.cuh (backward kernels.py:99-119, b = A conj(S)/|S|
// kernels.py:136-137, forward kernels.py:122-144) for np <= 112, with both
// complex GEMMs of a 128-row x 64-column tile issued as tcgen05.mma
// kind::tf32 (M = 128) and accumulated in TMEM:
//
//   backward  S[r][c] = sum_k V[r][k] X[c][k]   V = coef_k gy[r0+r][k] (A, TMEM)
//                                               X = gx[c0+c][k]        (B, smem)
//   b         = A conj(S)/|S| -> TMEM (A operand of the forward), phase write
//   forward   T[r][k] = sum_c b[r][c] X[c][k]   X^T staged c-contiguous (B, smem)
//   E_k       = sum_r gy[r0+r][k] T[r][k]       (CUDA cores, fixed-order reduce)
//
// FP32 accuracy from TF32 units: every operand is split x = hi + lo with
// hi = rna_tf32(x), and each real product is hi*hi + hi*lo + lo*hi (the
// dropped lo*lo term is ~2^-22 relative).  A complex MAC is four real
// products (Sr = Vr Xr - Vi Xi: the minus via the instruction's a_negate
// bit), so one 8-deep k-step is 12 MMAs per accumulator pair.
//
// TMEM (512 columns, lane = tile row):
//   [0, 128)    V' slots (2 x {Vr_h, Vr_l, Vi_h, Vi_l} x 16 spots)   backward
//   [0, 256)    b'  {br_h, br_l, bi_h, bi_l} x 64 columns            forward
//   [256, 384)  S = {Sr, Si} x 64 columns                            backward
//   [256, 256 + 2 NP)  T = {Tr, Ti} x NP spots                       forward
// Shared memory: two operand slots (a backward chunk of 16 spots x 64
// columns, or a forward chunk of 16 columns x NP spots, 4 planes each) in
// the SWIZZLE_NONE K-major canonical layout (8 x 16-byte core matrices),
// written by all threads while the previous chunk's MMAs run; one thread
// issues the MMAs and commits them to the slot's mbarrier.
//
// Encodings (instruction descriptor, shared-memory descriptor, TMEM
// st / ld, a_negate with A in TMEM) are checked by tools/umma_probe.cu.
#pragma once

#include "hs_kernels.cuh"
#include "hs_tile.cuh"

namespace hs {

constexpr int kUR = 128;         // tile rows (MMA M)
constexpr int kUC = 64;          // tile columns
constexpr int kUK = 16;          // spots per backward chunk / columns per forward chunk
constexpr int kUNPMax = 112;     // largest np (TMEM: 256 + 2 np <= 512)
constexpr int kUThreads = 256;
constexpr int kUSlot = 4 * kUNPMax * kUK * 4;  // 28 KB: forward chunk at np = 112

__host__ __device__ constexpr size_t hs_umma_smem_bytes()
{
    // 2 operand slots + 1 KB alignment + E reduce scratch [8 warps][64] float
    return 2 * (size_t)kUSlot + 1024 + 8 * 64 * sizeof(float);
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

__device__ __forceinline__ void hs_mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
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

template <int NP, bool WRITE>
__global__ void __launch_bounds__(kUThreads, 1) hs_umma_kernel(const TileArgs a)
{
    static_assert(NP % 16 == 0 && NP <= kUNPMax, "forward N = np must be a multiple of 16, <= 112");
    constexpr int NCC = kUC / kUK;           // forward chunks
    constexpr uint32_t BPL = kUC * kUK * 4;  // backward plane bytes (4 KB)
    constexpr uint32_t FPL = NP * kUK * 4;   // forward plane bytes
    constexpr uint32_t FLBO = (NP / 8) * 128;
    constexpr int KH = NP / 2;               // spots per thread in the E epilogue
    extern __shared__ __align__(1024) unsigned char smu[];
    __shared__ __align__(8) unsigned long long mbar[2];
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
    const float2 *gy = a.gy + (int64_t)pat * a.tab_stride;
    const int n = a.n;
    const int ksteps = (n + 7) / 8;          // backward k-steps (8 spots)
    const int nkc = (ksteps + 1) / 2;

    unsigned char *sbase = reinterpret_cast<unsigned char *>(((uintptr_t)smu + 1023) & ~(uintptr_t)1023);
    const uint32_t sb = hs_smem_addr(sbase);
    float *red = reinterpret_cast<float *>(sbase + 2 * kUSlot);  // [8][64]

    // ---- operand builders (all threads) ------------------------------------
    // backward chunk kc of X into byte offset `slot`: planes {Xr_h, Xr_l, Xi_h,
    // Xi_l}, [64 columns][16 spots] K-major: (c/8)*128 + (k/4)*1024 + (c%8)*16
    auto build_xb = [&](int kc, uint32_t slot) {
        const int c = tid >> 2, kq = tid & 3;
        const int gc = min(c0 + c, a.side - 1);
        const int k = kc * kUK + 4 * kq;
        const float4 *src = reinterpret_cast<const float4 *>(gx + (int64_t)gc * a.np + k);
        float4 u0 = __ldg(src), u1 = __ldg(src + 1);  // (k, k+1), (k+2, k+3)
        if (k >= n) u0 = make_float4(0.f, 0.f, 0.f, 0.f);  // table padding past n: zero
        if (k + 2 >= n) u1 = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 rh, rl, ih, il;
        hs_split4(u0.x, u0.z, u1.x, u1.z, rh, rl);
        hs_split4(u0.y, u0.w, u1.y, u1.w, ih, il);
        unsigned char *d = sbase + slot + (c >> 3) * 128 + kq * 1024 + (c & 7) * 16;
        *reinterpret_cast<float4 *>(d) = rh;
        *reinterpret_cast<float4 *>(d + BPL) = rl;
        *reinterpret_cast<float4 *>(d + 2 * BPL) = ih;
        *reinterpret_cast<float4 *>(d + 3 * BPL) = il;
    };
    // forward chunk cc of X^T: planes [NP spots][16 columns] K-major:
    // (k/8)*128 + (c/4)*FLBO + (k%8)*16 + (c%4)*4
    auto build_xf = [&](int cc, uint32_t slot) {
        const int cq = tid & 3;
        for (int k = tid >> 2; k < NP; k += kUThreads / 4) {
            float xr[4], xi[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int gc = min(c0 + cc * kUK + 4 * cq + j, a.side - 1);
                const float2 v = (k < n) ? __ldg(gx + (int64_t)gc * a.np + k) : make_float2(0.f, 0.f);
                xr[j] = v.x;
                xi[j] = v.y;
            }
            float4 rh, rl, ih, il;
            hs_split4(xr[0], xr[1], xr[2], xr[3], rh, rl);
            hs_split4(xi[0], xi[1], xi[2], xi[3], ih, il);
            unsigned char *d = sbase + slot + (k >> 3) * 128 + cq * FLBO + (k & 7) * 16;
            *reinterpret_cast<float4 *>(d) = rh;
            *reinterpret_cast<float4 *>(d + FPL) = rl;
            *reinterpret_cast<float4 *>(d + 2 * FPL) = ih;
            *reinterpret_cast<float4 *>(d + 3 * FPL) = il;
        }
    };

    build_xb(0, 0);  // gx: an input of the whole solve
    // -- below: the previous pass's results (status, coef); TMEM is taken
    // only now, so a dependent-launched CTA never holds it while waiting
    hs_pdl_wait_prev();
    if (a.f.u.status[pat] != 0) return;  // uniform per CTA
    if (tid < NP) coef_s[tid] = (tid < n) ? a.coef[(int64_t)pat * a.np + tid] : make_float2(0.f, 0.f);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(hs_smem_addr(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(hs_smem_addr(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(hs_smem_addr(&mbar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    hs_tc_fence_before();
    __syncthreads();
    hs_tc_fence_after();
    const uint32_t tm = s_tmem;
    const uint32_t tl = tm + ((uint32_t)(32 * q) << 16);  // this warp's lane quarter
    const uint32_t bar0 = hs_smem_addr(&mbar[0]), bar1 = hs_smem_addr(&mbar[1]);
    uint32_t ph0 = 0, ph1 = 0;
    bool pend0 = false, pend1 = false;
    auto wait_slot = [&](int s) {
        if (s == 0 && pend0) { hs_mbar_wait(bar0, ph0); ph0 ^= 1; pend0 = false; }
        if (s == 1 && pend1) { hs_mbar_wait(bar1, ph1); ph1 ^= 1; pend1 = false; }
        hs_tc_fence_after();
    };
    auto commit_slot = [&](int s) {  // tid 0 issued the MMAs; every thread tracks the phase
        if (tid == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             s ? bar1 : bar0)
                         : "memory");
        if (s) pend1 = true; else pend0 = true;
    };
    // operands written by this thread (smem via the generic proxy, TMEM via
    // tcgen05.st) become visible to the MMA-issuing thread
    auto publish = [&]() {
        hs_tc_wait_st();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        hs_tc_fence_before();
        __syncthreads();
        hs_tc_fence_after();
    };

    const int grow = r0 + row;
    const bool row_in = grow < a.side;
    const float2 *gyrow = gy + (int64_t)min(grow, a.side - 1) * a.np;

    // ---- backward -------------------------------------------------------------
    constexpr uint32_t TS = 256;            // S / T column base
    const uint32_t idb = hs_idesc_tf32(kUC, false), idbn = hs_idesc_tf32(kUC, true);
    for (int kc = 0; kc < nkc; ++kc) {
        const int s = kc & 1;
        wait_slot(s);  // chunk kc - 2 (same slot) consumed
        if (kc > 0) build_xb(kc, s * (4 * BPL));
        {   // V' for spots kc*16 + 8h .. +8 of this thread's row into TMEM slot s
            float vr[8], vi[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = kc * kUK + 8 * h + j;
                const float2 g = row_in ? __ldg(gyrow + k) : make_float2(0.f, 0.f);
                const float2 w = coef_s[k];
                vr[j] = fmaf(w.x, g.x, -w.y * g.y);
                vi[j] = fmaf(w.x, g.y, w.y * g.x);
            }
            float p[8];
            const uint32_t col = tl + s * 64 + 8 * h;
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = hs_tf32_hi(vr[j]);
            hs_tc_st8(col, p);
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = vr[j] - hs_tf32_hi(vr[j]);
            hs_tc_st8(col + 16, p);
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = hs_tf32_hi(vi[j]);
            hs_tc_st8(col + 32, p);
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = vi[j] - hs_tf32_hi(vi[j]);
            hs_tc_st8(col + 48, p);
        }
        publish();
        if (tid == 0) {
            const uint32_t xs = sb + s * (4 * BPL);
            for (int ks = 0; ks < 2 && kc * 2 + ks < ksteps; ++ks) {
                const uint32_t va = tm + s * 64 + ks * 8;  // Vr_h; +16 Vr_l, +32 Vi_h, +48 Vi_l
                const uint32_t xo = xs + ks * 2 * 1024;
                const uint64_t xrh = hs_sdesc(xo, 1024, 128), xrl = hs_sdesc(xo + BPL, 1024, 128);
                const uint64_t xih = hs_sdesc(xo + 2 * BPL, 1024, 128), xil = hs_sdesc(xo + 3 * BPL, 1024, 128);
                const uint32_t acc = (kc | ks) ? 1u : 0u;
                const uint32_t sr = tm + TS, si = tm + TS + kUC;
                hs_mma_ts(sr, va, xrh, idb, acc);
                hs_mma_ts(sr, va, xrl, idb, 1);
                hs_mma_ts(sr, va + 16, xrh, idb, 1);
                hs_mma_ts(sr, va + 32, xih, idbn, 1);
                hs_mma_ts(sr, va + 32, xil, idbn, 1);
                hs_mma_ts(sr, va + 48, xih, idbn, 1);
                hs_mma_ts(si, va, xih, idb, acc);
                hs_mma_ts(si, va, xil, idb, 1);
                hs_mma_ts(si, va + 16, xih, idb, 1);
                hs_mma_ts(si, va + 32, xrh, idb, 1);
                hs_mma_ts(si, va + 32, xrl, idb, 1);
                hs_mma_ts(si, va + 48, xrh, idb, 1);
            }
        }
        commit_slot(s);
    }
    wait_slot(0);
    wait_slot(1);

    // ---- b = A conj(S)/|S| into TMEM b' (columns 32h .. 32h+32 of the row) --
    const int64_t prow = (int64_t)min(grow, a.side - 1) * a.side;
#pragma unroll 1
    for (int cb = 0; cb < 32; cb += 8) {
        const int cl = 32 * h + cb;  // tile column of element 0
        float sr[8], si[8], p[8];
        hs_tc_ld8(tl + TS + cl, sr);
        hs_tc_ld8(tl + TS + kUC + cl, si);
        hs_tc_wait_ld();
        float br[8], bi[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = c0 + cl + j;
            const bool in = row_in && c < a.side;
            const float A = in ? __ldg(a.amp_img + prow + c) : 0.f;
            hs_bvec_exact(sr[j], si[j], A, br[j], bi[j]);
            if (WRITE && in) {
                const int32_t di = __ldg(a.idx_img + prow + c);
                if (di >= 0) {
                    const double ph = hs_phase_f64(sr[j], si[j]);
                    a.phase_out[(int64_t)pat * a.phase_stride + di] = ph;
                    if (a.raster) a.raster[(int64_t)pat * a.side * a.side + prow + c] = hs_gray_linear(ph);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = hs_tf32_hi(br[j]);
        hs_tc_st8(tl + cl, p);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = br[j] - hs_tf32_hi(br[j]);
        hs_tc_st8(tl + 64 + cl, p);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = hs_tf32_hi(bi[j]);
        hs_tc_st8(tl + 128 + cl, p);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = bi[j] - hs_tf32_hi(bi[j]);
        hs_tc_st8(tl + 192 + cl, p);
    }

    // ---- forward ---------------------------------------------------------------
    const uint32_t idf = hs_idesc_tf32(NP, false), idfn = hs_idesc_tf32(NP, true);
    for (int cc = 0; cc < NCC; ++cc) {
        const int s = cc & 1;
        wait_slot(s);
        build_xf(cc, s * kUSlot);
        publish();  // (cc = 0: also b' and the S reads before T overwrites S)
        if (tid == 0) {
            const uint32_t xs = sb + s * kUSlot;
            for (int cs = 0; cs < 2; ++cs) {
                const uint32_t ba = tm + cc * kUK + cs * 8;  // br_h; +64 br_l, +128 bi_h, +192 bi_l
                const uint32_t xo = xs + cs * 2 * FLBO;
                const uint64_t xrh = hs_sdesc(xo, FLBO, 128), xrl = hs_sdesc(xo + FPL, FLBO, 128);
                const uint64_t xih = hs_sdesc(xo + 2 * FPL, FLBO, 128), xil = hs_sdesc(xo + 3 * FPL, FLBO, 128);
                const uint32_t acc = (cc | cs) ? 1u : 0u;
                const uint32_t tr = tm + TS, ti = tm + TS + NP;
                hs_mma_ts(tr, ba, xrh, idf, acc);
                hs_mma_ts(tr, ba, xrl, idf, 1);
                hs_mma_ts(tr, ba + 64, xrh, idf, 1);
                hs_mma_ts(tr, ba + 128, xih, idfn, 1);
                hs_mma_ts(tr, ba + 128, xil, idfn, 1);
                hs_mma_ts(tr, ba + 192, xih, idfn, 1);
                hs_mma_ts(ti, ba, xih, idf, acc);
                hs_mma_ts(ti, ba, xil, idf, 1);
                hs_mma_ts(ti, ba + 64, xih, idf, 1);
                hs_mma_ts(ti, ba + 128, xrh, idf, 1);
                hs_mma_ts(ti, ba + 128, xrl, idf, 1);
                hs_mma_ts(ti, ba + 192, xrh, idf, 1);
            }
        }
        commit_slot(s);
    }
    wait_slot(0);
    wait_slot(1);

    // ---- E_k = sum_r gy[r][k] T[r][k]: spots KH h .. KH (h+1) of the row in
    // two 8-aligned parts (KA + KB = KH, KA <= 32); each part is
    // transpose-reduced over the warp's 32 rows (64 padded values -> 2 per
    // lane), then the 4 lane-quarter warps are summed in order through shared
    // memory.
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
                float tr[8], ti[8];
                const int kk = kbase + 8 * k8;
                hs_tc_ld8(tl + TS + kk, tr);
                hs_tc_ld8(tl + TS + NP + kk, ti);
                hs_tc_wait_ld();
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float2 g = row_in ? __ldg(gyrow + kk + j) : make_float2(0.f, 0.f);
                    v[16 * k8 + 2 * j] = fmaf(g.x, tr[j], -g.y * ti[j]);
                    v[16 * k8 + 2 * j + 1] = fmaf(g.x, ti[j], g.y * tr[j]);
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
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    if (a.f.u.act != ACT_NONE) hs_fold(a.f, pat, tile, reinterpret_cast<char *>(sbase));
}

typedef void (*UmmaFn)(TileArgs);
UmmaFn hs_select_umma(int np, bool write);

}  // namespace hs
