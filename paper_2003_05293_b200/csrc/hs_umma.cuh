// hs_umma.cuh -- full-range fused pass on the tcgen05 tensor cores.
//
// Same pass as hs_tile.cuh (backward kernels.py:99-119, b = A conj(S)/|S|
// kernels.py:136-137, forward kernels.py:122-144) -- selected for 32 < n <=
// 128 (hs_plan.cu tile_set) -- with both complex GEMMs of a 128-row x
// 64-column tile issued as tcgen05.mma kind::tf32 (M = 128) and accumulated
// in TMEM:
//
//   backward  S[r][c] = sum_k gy[r0+r][k] X'[c][k]   gy planes (A, smem, TMA)
//                                                    X' = coef_k gx[c0+c][k] (B, smem)
//   b         = A conj(S)/|S| (registers), phase write
//   forward   T[r][k] = sum_c b[r][c] X[c][k]   b (A, smem), X^T (B, smem)
//   E_k       = sum_r gy[r0+r][k] T[r][k]       (CUDA cores, fixed-order reduce)
//
// FP32 accuracy from TF32 units: every operand is split x = hi + lo with
// hi = rna_tf32(x), and each real product is hi*hi + hi*lo + lo*hi (the
// dropped lo*lo term is ~2^-22 relative).  Backward: one N = 128 MMA
// produces [Sr | Si] from the stacked B planes [Xr; Xi] and [-Xi; Xr], so a
// complex 8-deep k-step is 6 MMAs (A in {gr, gi} x 3 split terms).  Forward:
// Tr and Ti are separate N = np MMAs (the minus via the a_negate bit), 12 per
// k-step.
//
// Two CTAs per SM (256 TMEM columns each), so one CTA's CUDA-core phases
// (operand builds, b, the E reduce, the fold) overlap the other's MMAs:
//   TMEM [0, 128)     S = {Sr, Si} x 64 columns                            backward
//        [0, 2 NP)    T = {Tr, Ti} x NP spots                              forward
// (np = 128 runs the spot-chunked variant NP = 128: T fills all 256 columns,
// one CTA per SM, the backward's k-steps summed in groups in registers.)
// S is read once into registers (b: 32 columns per thread), which frees the
// columns T reuses.  The operands that do not change between passes are
// written once per table build by hs_umma_prep_kernel as hi/lo planes (fp16)
// already in the shared-memory operand layout -- gy (A of the backward,
// [band][k-step] blocks of 16 KB) and X^T (B of the forward, 8-column blocks
// of <= 16 KB) -- and each k-step's block is one TMA bulk copy, issued one
// step ahead; the per-pass coefficients go on the B side of the backward
// (X' = coef_k gx[c][k], built by warps 4-7) and b' (A of the forward) is
// written by every thread for its row.  The E epilogue reads gy in fp32
// from a row-coalesced copy written beside the planes.  Shared memory: A and
// B rings (3 slots of 16 KB at two CTAs per SM; 6 for the spot-chunked
// variant at one CTA per SM), SWIZZLE_NONE K-major canonical layout (8 x
// 16-byte core matrices).
//
// Roles per k-step j: the threads that write operands (warps 4-7 in the
// backward, all warps in the forward) fence them into the async proxy and
// arrive, one elected lane per warp, on operand barrier j % R; warp 1's
// lane 0 issues the TMA of step j + 1 as one more arrival on that barrier
// (expect_tx) after MMA(j + 1 - R) has freed the slot; the converged warp 0
// waits once for the barrier and issues the step's MMAs and commit with
// elect.sync (from a one-thread branch the compiler wrapped every MMA in an
// ELECT / R2UR / BRA.U.ANY loop, ~100 cycles each).  Slots are reused R - 1
// steps later, so up to R - 1 steps of MMAs are in flight.
//
// Per-CTA timeline (HS_UMMA_TRACE=1 with hs_time_kernel: clock64 at fixed
// points of one CTA; round 2 final).  B = 32, np = 112, two CTAs per SM:
// prologue 2.6k cycles, 7 backward k-steps ~2k each, b 8.4k, 4 forward
// k-steps ~1.7k, E epilogue 12.2k, fold 3.8k (52k per tile, two tiles
// overlapping per SM).  Config 4 (np = 1008, one CTA per SM): 63 backward
// k-steps ~1.5k each (was 2.1k before the issue changes above), then 8
// forward spot chunks.  Tensor pipe ~25-28% active (ncu): the cadence is
// the issue chain (barrier wait, descriptor moves to uniform registers,
// 6-12 MMA issues, commit) and, per tile, the CUDA-core phases (b, E).
//
// Encodings (instruction descriptor, shared-memory descriptor, TMEM
// st / ld, a_negate) are checked by tools/umma_probe.cu.
#pragma once

#include <cuda_fp16.h>

#include "hs_kernels.cuh"
#include "hs_tile.cuh"

namespace hs {

constexpr int kUR = 128;         // tile rows (MMA M)
constexpr int kUC = 64;          // tile columns
// Operand format.  kind::f16 (default): every operand is split x = hi + lo
// into two fp16 values and each real product is hi*hi + hi*lo + lo*hi, fp32
// accumulate -- 22-bit products like the tf32 split, but an f16 MMA has
// twice the K of a tf32 MMA at the same cost: a shared-memory-operand MMA
// takes ~118 cycles for N <= 128 either way (tools/mma_rate.cu), so the
// MMA time per tile halves.  The fp16 lo of a value below 2^-2 is subnormal;
// the split then keeps an absolute error <= 2^-25, against unit-scale
// phasors and |S| ~ sum a_n that is below the fp32 pixel noise.
// HS_UMMA_F16=0 builds the tf32 variant.
#ifndef HS_UMMA_F16
#define HS_UMMA_F16 1
#endif
constexpr bool kF16 = HS_UMMA_F16 != 0;
constexpr int kUEB = kF16 ? 2 : 4;  // operand element bytes
constexpr int kUF = 32 / kUEB;      // spots / columns per stage (one MMA k-step: 32 bytes of K)
constexpr int kUQ = 16 / kUEB;      // elements per 16-byte core-matrix row
constexpr int kUNPMax = 112;     // largest np run as one forward spot chunk (N = np)
constexpr int kUNPC = 128;       // forward spot chunk for larger np (T: 2 x 128 TMEM columns)
constexpr int kUThreads = 256;
constexpr int kUTmem = 256;      // TMEM columns per CTA (two CTAs per SM)
#ifndef HS_UMMA_RING
#define HS_UMMA_RING 3
#endif
// The spot-chunked variant (np > 112) runs one CTA per SM, whose shared
// memory holds deeper rings: more k-steps of MMAs in flight (a k-step's
// MMAs take ~2.6k cycles from issue to completion, four times their
// tensor-pipe time, so two in flight leave the pipe idle).
#ifndef HS_UMMA_RING_CH
#define HS_UMMA_RING_CH 6
#endif
// ring depth (A ring: gy planes (backward, TMA) / b' (forward, threads);
// B ring: X' (backward, threads) / X^T planes (forward, TMA))
__host__ __device__ constexpr int hs_umma_ring(int np) { return np <= 112 ? HS_UMMA_RING : HS_UMMA_RING_CH; }
constexpr int kUA = HS_UMMA_RING;  // ring of the np <= 112 variants
constexpr int kUD = 1;             // TMA prefetch distance (steps ahead of the MMA issue)
constexpr int kUMinBlocks = kUA <= 3 ? 2 : 1;  // CTAs per SM the shared memory allows
constexpr int kUAPl = kUR * 32;                     // A plane [128 rows][32 bytes of K] (4 KB)
constexpr int kUASlot = 4 * kUAPl;                  // 16 KB
// B slot: the backward's stacked X' planes ([Xr; Xi] and [-Xi; Xr], 128 rows,
// 16 KB) or the X^T of one forward k-step (npc spots, <= 16 KB).
__host__ __device__ constexpr int hs_umma_bslot(int) { return 4 * 2 * kUC * 32; }

__host__ __device__ constexpr size_t hs_umma_smem_bytes(int np)
{
    // rings + 128 B alignment slack + E reduce scratch [4 groups][8 warps][32] float + coef [np]
    return (size_t)hs_umma_ring(np) * (kUASlot + hs_umma_bslot(np <= kUNPMax ? np : kUNPC)) + 128 +
           4 * 8 * 32 * sizeof(float) + 8 * (size_t)np;
}

// Forward spot chunk (the MMA N) and chunk count for a table width np:
// one chunk of np spots up to 112, else chunks of 128 (the last zero-padded).
__host__ __device__ constexpr int hs_umma_npc(int np) { return np <= kUNPMax ? np : kUNPC; }
__host__ __device__ constexpr int hs_umma_nsc(int np) { return (np + hs_umma_npc(np) - 1) / hs_umma_npc(np); }

// Operand planes of one pattern (constant per table build):
//   gy : [band][k-step][4][128 rows][kUF spots]                      (A of the backward)
//   X^T: [column block of kUF][spot chunk][4][npc spots][kUF columns] (B of the forward),
//        ceil(side / kUF) + kUC / kUF column blocks (the tail blocks are zero)
__host__ __device__ constexpr int64_t hs_umma_gy_floats(int side, int np)
{
    return (int64_t)((side + kUR - 1) / kUR) * (np / kUF) * (kUASlot / 4);
}
__host__ __device__ constexpr int hs_umma_xblocks(int side) { return (side + kUF - 1) / kUF + kUC / kUF; }
__host__ __device__ constexpr int64_t hs_umma_xblock_floats(int np)
{
    return (int64_t)hs_umma_nsc(np) * 4 * hs_umma_npc(np) * 8;  // 4 planes x npc rows x 32 bytes
}
// gy in fp32 for the E epilogue: [band][8-spot block][4][128 rows] float4
// (re of spots 0-3, im 0-3, re 4-7, im 4-7): a thread (row) reads 4
// coalesced float4 per 8 spots, no operand-format decode
__host__ __device__ constexpr int64_t hs_umma_gye_floats(int side, int np)
{
    return (int64_t)((side + kUR - 1) / kUR) * np * 4 * kUR / 2;
}
__host__ __device__ constexpr int64_t hs_umma_plane_floats(int side, int np)
{
    return hs_umma_gy_floats(side, np) + (int64_t)hs_umma_xblocks(side) * hs_umma_xblock_floats(np) +
           hs_umma_gye_floats(side, np);
}
// grid.x of hs_umma_prep_kernel
__host__ __device__ constexpr int hs_umma_prep_blocks(int side, int np)
{
    return (side + kUR - 1) / kUR * (np / kUF) + hs_umma_xblocks(side) * hs_umma_nsc(np) +
           (side + kUR - 1) / kUR * (np / 8);
}

// Byte offset of element (r, k) in a [128 rows][kUF] K-major operand plane
// (SWIZZLE_NONE core matrices: 8 rows x 16 bytes; K halves 2048 B apart).
__host__ __device__ constexpr int hs_uoffb(int r, int k) { return r * 16 + (k / kUQ) * 2048 + (k % kUQ) * kUEB; }

// hi/lo split of one value in the operand format; returns the raw bits
__device__ __forceinline__ void hs_split1(float v, uint32_t &hb, uint32_t &lb)
{
    if constexpr (kF16) {
        const __half h = __float2half_rn(v);
        const __half l = __float2half_rn(v - __half2float(h));
        hb = __half_as_ushort(h);
        lb = __half_as_ushort(l);
    } else {
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(v - __uint_as_float(hb)));
    }
}

// fp16 hi/lo split of two values into packed words (v0 in the low half):
// one paired conversion each way, bitwise the same as two hs_split1
__device__ __forceinline__ void hs_split2(float v0, float v1, uint32_t &h, uint32_t &l)
{
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(v1), "f"(v0));  // d.hi = cvt(a), d.lo = cvt(b)
    const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&h));
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(v1 - f.y), "f"(v0 - f.x));
}

__device__ __forceinline__ void hs_put(unsigned char *p, uint32_t bits)
{
    if constexpr (kF16) *reinterpret_cast<unsigned short *>(p) = (unsigned short)bits;
    else *reinterpret_cast<uint32_t *>(p) = bits;
}

__device__ __forceinline__ void hs_split_store(float v, unsigned char *dst, int plane_bytes)
{
    uint32_t h, l;
    hs_split1(v, h, l);
    hs_put(dst, h);
    hs_put(dst + plane_bytes, l);
}

// hi/lo split of one 16-byte core-matrix row chunk (kUQ values), and its negation
__device__ __forceinline__ void hs_split_chunk(const float *v, uint4 &hi, uint4 &lo)
{
    if constexpr (kF16) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) hs_split2(v[2 * i], v[2 * i + 1], hw[i], lw[i]);
        hi = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        lo = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    } else {
        uint32_t hb[kUQ], lb[kUQ];
#pragma unroll
        for (int i = 0; i < kUQ; ++i) hs_split1(v[i], hb[i], lb[i]);
        hi = make_uint4(hb[0], hb[1], hb[2], hb[3]);
        lo = make_uint4(lb[0], lb[1], lb[2], lb[3]);
    }
}
__device__ __forceinline__ uint4 hs_neg_chunk(uint4 v)
{
    constexpr uint32_t m = kF16 ? 0x80008000u : 0x80000000u;
    return make_uint4(v.x ^ m, v.y ^ m, v.z ^ m, v.w ^ m);
}

// operand element -> float (the gy planes read back by the E epilogue)
__device__ __forceinline__ float hs_opnd(uint32_t bits)
{
    if constexpr (kF16) return __half2float(__ushort_as_half((unsigned short)bits));
    else return __uint_as_float(bits);
}

// gy / gx -> tf32 hi/lo planes {re_h, re_l, im_h, im_l} in the operand
// layouts.  grid (bands * np / 8 + xblocks * nsc, B), 256 threads.
static __global__ void hs_umma_prep_kernel(const float2 *__restrict__ gx, const float2 *__restrict__ gy,
                                           float *__restrict__ planes, int side, int np, int64_t tab_stride,
                                           int64_t plane_stride)
{
    const int nks = np / kUF;
    const int ngy = (side + kUR - 1) / kUR * nks;
    const int pat = blockIdx.y;
    unsigned char *base = reinterpret_cast<unsigned char *>(planes + (int64_t)pat * plane_stride);
    if ((int)blockIdx.x < ngy) {
        const int band = blockIdx.x / nks, ks = blockIdx.x % nks;
        unsigned char *dst = base + (int64_t)blockIdx.x * kUASlot;
        for (int i = threadIdx.x; i < kUR * kUF; i += blockDim.x) {
            const int r = i / kUF, k = i % kUF;
            const int grow = band * kUR + r;
            const float2 v = grow < side ? gy[(int64_t)pat * tab_stride + (int64_t)grow * np + ks * kUF + k]
                                         : make_float2(0.f, 0.f);
            const int o = hs_uoffb(r, k);
            hs_split_store(v.x, dst + o, kUAPl);
            hs_split_store(v.y, dst + o + 2 * kUAPl, kUAPl);
        }
    } else if ((int)blockIdx.x >= ngy + hs_umma_xblocks(side) * hs_umma_nsc(np)) {
        const int e = blockIdx.x - ngy - hs_umma_xblocks(side) * hs_umma_nsc(np);  // band * np / 8 + block
        const int band = e / (np / 8), blk = e % (np / 8);
        float4 *dst = reinterpret_cast<float4 *>(planes + (int64_t)pat * plane_stride + hs_umma_gy_floats(side, np) +
                                                 (int64_t)hs_umma_xblocks(side) * hs_umma_xblock_floats(np)) +
                      (int64_t)e * 4 * kUR;
        for (int i = threadIdx.x; i < 4 * kUR; i += blockDim.x) {
            const int qd = i / kUR, r = i % kUR;  // quad qd: spots 4 (qd / 2) .., re (qd even) / im
            const int grow = band * kUR + r;
            float v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 g = grow < side ? gy[(int64_t)pat * tab_stride + (int64_t)grow * np + blk * 8 + 4 * (qd >> 1) + j]
                                             : make_float2(0.f, 0.f);
                v[j] = (qd & 1) ? g.y : g.x;
            }
            dst[qd * kUR + r] = make_float4(v[0], v[1], v[2], v[3]);
        }
    } else {
        const int nsc = hs_umma_nsc(np), npc = hs_umma_npc(np);
        const int cb = (blockIdx.x - ngy) / nsc, sc = (blockIdx.x - ngy) % nsc;
        const int pl = npc * 32;  // plane bytes
        unsigned char *dst = base + 4 * hs_umma_gy_floats(side, np) + (int64_t)(blockIdx.x - ngy) * 4 * pl;
        for (int i = threadIdx.x; i < npc * kUF; i += blockDim.x) {
            const int k = i / kUF, c = i % kUF;
            const int gc = cb * kUF + c, gk = sc * npc + k;
            const float2 v = (gc < side && gk < np) ? gx[(int64_t)pat * tab_stride + (int64_t)gc * np + gk]
                                                    : make_float2(0.f, 0.f);
            // K-major over columns: 8-spot groups 128 B apart (SBO), column halves at npc/8 * 128 (LBO)
            const int o = (k >> 3) * 128 + (c / kUQ) * (npc / 8) * 128 + (k & 7) * 16 + (c % kUQ) * kUEB;
            hs_split_store(v.x, dst + o, pl);
            hs_split_store(v.y, dst + o + 2 * pl, pl);
        }
    }
}

// ---- PTX wrappers --------------------------------------------------------
__device__ __forceinline__ uint64_t hs_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);  // sm100 version, no swizzle
}

// kind::tf32 (A/B format 2) or kind::f16 (fp16: format 0), f32 accumulate,
// A and B K-major
__host__ __device__ constexpr uint32_t hs_idesc_tf32(int n, bool neg)
{
    return (1u << 4) | ((kF16 ? 0u : 2u) << 7) | ((kF16 ? 0u : 2u) << 10) | ((neg ? 1u : 0u) << 13) |
           ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kUR >> 4) << 24);
}

// A from TMEM
__device__ __forceinline__ void hs_mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    if constexpr (kF16)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                     "r"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                     "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

// A from shared memory.  Called by a whole converged warp with warp-uniform
// operands; one elected lane issues (the operands stay in uniform
// registers -- issued from a one-thread branch, every MMA was wrapped in an
// ELECT / R2UR / BRA.U.ANY loop, ~100 cycles each).
__device__ __forceinline__ void hs_mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    if constexpr (kF16)
        asm volatile("{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                     "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        asm volatile("{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
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
// (lo is rounded to tf32 as well: the tensor core would otherwise truncate
// its low mantissa bits, a bias that grows linearly in long sums)
__device__ __forceinline__ void hs_split4(float a, float b, float c, float d, float4 &hi, float4 &lo)
{
    hi = make_float4(hs_tf32_hi(a), hs_tf32_hi(b), hs_tf32_hi(c), hs_tf32_hi(d));
    lo = make_float4(hs_tf32_hi(a - hi.x), hs_tf32_hi(b - hi.y), hs_tf32_hi(c - hi.z), hs_tf32_hi(d - hi.w));
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

template <int NP, int WRITE>  // WRITE: 0 no phase, 1 f64 phases, 2 4-byte phase codes
__global__ void __launch_bounds__(kUThreads, NP == kUNPC ? 1 : kUMinBlocks) hs_umma_kernel(const TileArgs a)
{
    static_assert(NP % 16 == 0 && (NP <= kUNPMax || NP == kUNPC), "forward N: np <= 112 or chunks of 128");
    constexpr int NCC = kUC / kUF;           // forward k-steps (4 fp16 / 8 tf32)
    constexpr int NG8 = kUC / 8;             // 8-column groups of a tile row (b phase)
    constexpr uint32_t FPL = NP * 32;        // forward X^T plane bytes (= floats of one 4-plane block)
    constexpr uint32_t FLBO = (NP / 8) * 128;
    constexpr int KH = NP / 2;               // spots per thread in the E epilogue
    constexpr int kUBSlot = hs_umma_bslot(NP);
    constexpr int RA = hs_umma_ring(NP), RB = RA;  // ring slots
    constexpr int RW = RA - kUD;  // MMA wait distance: step j reuses the slots of step j - RW
    extern __shared__ __align__(128) unsigned char smu[];
    // MMA done [0, 4), A full (gy TMA) [4, 8), B full (X^T TMA) [8, 11),
    // operands written (all threads arrive) [11, 15)
    __shared__ __align__(8) unsigned long long mbar[3 * RA + RB];
    __shared__ uint32_t s_tmem;

    hs_pdl_launch_next();
    const int pat = blockIdx.y;
    const int tile = a.f.chunk_base + blockIdx.x;
    // timing probe: clock64 at fixed points of one CTA (tile 100, pattern 0)
    const bool trc = a.trace && blockIdx.x == 100 && blockIdx.y == 0;
    auto TR = [&](int who, int slot) {
#if HS_PROBES
        if (trc && (int)threadIdx.x == who) a.trace[slot] = clock64();
#else
        (void)trc, (void)who, (void)slot;
#endif
    };
    TR(0, 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = warp & 3, h = warp >> 2;  // TMEM lane quarter, column / spot half
    const int row = 32 * q + lane;          // tile row of this thread (TMEM lane)
    const int packed = __ldg(a.tiles + tile);
    const int r0 = packed >> 16, c0 = packed & 0xffff;  // c0: multiple of kUF
    const float2 *gx = a.gx + (int64_t)pat * a.tab_stride;
    const float *pbase = a.gyp + (int64_t)pat * a.gyp_stride;
    const float *gyp = pbase + (int64_t)(r0 / kUR) * (a.np / kUF) * (kUASlot / 4);
    // forward spot chunks of NP: one when np <= 112 (b dies before the E
    // reduce); chunks of 128 otherwise (b stays live: one CTA per SM, no spills)
    const int nsc = NP <= kUNPMax ? 1 : hs_umma_nsc(a.np);
    const float *xtp = pbase + hs_umma_gy_floats(a.side, a.np) + (int64_t)(c0 / kUF) * nsc * FPL;
    const int n = a.n;
    const int ksteps = (n + kUF - 1) / kUF;  // backward k-steps (kUF spots)
    const int nsteps = ksteps + nsc * NCC;   // step sequence: backward, then forward per spot chunk

    unsigned char *sbase = reinterpret_cast<unsigned char *>(((uintptr_t)smu + 127) & ~(uintptr_t)127);
    const uint32_t sb = hs_smem_addr(sbase);
    const uint32_t sa = sb, sbb = sb + RA * kUASlot;  // A ring, B ring
    float *red = reinterpret_cast<float *>(sbase + RA * kUASlot + RB * kUBSlot);  // [4][8][32]
    float2 *coef_s = reinterpret_cast<float2 *>(red + 4 * 8 * 32);                  // [np]
    const int grow = r0 + row;
    const bool row_in = grow < a.side;

    // ---- backward X' loads: thread (column c = tid % 64, K half kq =
    // (tid / 64) % 2) of warps 4-7 loads the kUQ spots kUF ks + kUQ kq .. of
    // gx[c0 + c]; two k-steps in flight.  A warp's 32 threads hold 32
    // consecutive columns of one K half, so each of its X' plane stores
    // is 512 contiguous bytes (4 wavefronts, no bank conflicts)
    const bool xb_on = tid >= kUThreads - 2 * kUC;  // warps 4-7 (warp 0 issues the MMAs)
    const int xb_c = tid & (kUC - 1), xb_kq = (tid >> 6) & 1;
    const float4 *xb_src = reinterpret_cast<const float4 *>(gx + (int64_t)min(c0 + xb_c, a.side - 1) * a.np);
    constexpr int XV = kUQ / 2;  // float4 (two complex) per thread and k-step
    float4 xn[XV];               // gx of the next k-step to build
    auto load_b = [&](int ks, float4 (&d)[XV]) {
        if (xb_on && ks < ksteps) {
            const int k = ks * kUF + kUQ * xb_kq;
#pragma unroll
            for (int i = 0; i < XV; ++i) d[i] = __ldg(xb_src + k / 2 + i);
        }
    };
    load_b(0, xn);  // gx: an input of the whole solve

    // -- below: the previous pass's results (status, coef); TMEM is taken
    // only now, so a dependent-launched CTA never holds it while waiting
    hs_pdl_wait_prev();
    if (a.f.u.status[pat] != 0) return;  // uniform per CTA
    // coef past n is zero (the seed writes the whole np row, hs_update only k < n)
    for (int k = tid; k < a.np; k += kUThreads) coef_s[k] = a.coef[(int64_t)pat * a.np + k];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(hs_smem_addr(&s_tmem)),
                     "n"(NP == kUNPC ? 2 * kUTmem : kUTmem));  // spot-chunked: 512 (double-buffered T)
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const uint32_t bar = hs_smem_addr(&mbar[0]);
    const uint32_t bar_op = bar + 8 * (2 * RA + RB);
    auto bulk = [](uint32_t dst, const float *src, uint32_t bytes, uint32_t fb) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         dst),
                     "l"(src), "r"(bytes), "r"(fb)
                     : "memory");
    };
    // (warp 1) gy planes of backward step j -> A slot j % RA, X^T planes of
    // forward step j -> B slot j % RB, kUD steps ahead, issued at step i after
    // the wait for MMA(i - RW).  The copy is one more arrival (with its byte
    // count) on step j's operand barrier, so thread 0 waits once per step for
    // the threads' operands and the TMA together.
    auto tma_ahead = [&](int i) {
        const int j = i + kUD;
        if (j < ksteps) {
            bulk(sa + (j % RA) * kUASlot, gyp + (int64_t)j * (kUASlot / 4), kUASlot, bar_op + 8 * (j % RA));
        } else if (j < nsteps) {
            const int f = j - ksteps;  // spot chunk f / 8, column block f % 8
            bulk(sbb + (j % RB) * kUBSlot, xtp + ((int64_t)(f % NCC) * nsc + f / NCC) * FPL, 4 * FPL,
                 bar_op + 8 * (j % RA));
        }
    };
    if (tid == 0) {
        for (int i = 0; i < 2 * RA + RB; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8 * i));
        for (int i = 0; i < RA; ++i)  // one (elected) arrival per warp + the step's TMA
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_op + 8 * i), "n"(kUThreads / 32 + 1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = -kUD; i < 0; ++i) tma_ahead(i);  // steps 0 .. kUD-1
    }
    hs_tc_fence_before();
    __syncthreads();
    hs_tc_fence_after();
    TR(0, 1);
    const uint32_t tm = s_tmem;
    const uint32_t tl = tm + ((uint32_t)(32 * q) << 16);  // this warp's lane quarter

    // MMA completion of step j is completion (j / 4) of barrier j % 4; waits
    // happen in order, never two phases behind.
    int done = 0;  // steps known complete
    auto wait_mma = [&](int j) {
        for (; done <= j; ++done) hs_mbar_wait(bar + 8 * (done % RA), (uint32_t)(done / RA) & 1u);
        hs_tc_fence_after();
    };
    auto commit = [&](int j) {  // thread 0, after issuing step j's MMAs
        asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
                         bar + 8 * (j % RA))
                     : "memory");
    };
    // Step j's operands written by the threads (generic proxy; TMEM reads
    // retired) become visible to the MMA-issuing thread (async proxy): every
    // thread arrives on operand barrier j % 4 (completion j / 4), thread 0
    // waits for it.  No CTA-wide barrier per step: the other warps run ahead
    // until the MMA-done wait two steps back.
    // Each thread fences its own writes into the async proxy; the warp
    // converges and one lane arrives for it (256 single-thread arrivals on
    // one barrier word serialised into ~1k cycles per step).
    // Backward steps (bwd): warp 0 -- the issuing thread's own warp, which
    // writes no operand -- does not arrive; warp 1 arrives for it (count 2).
    // At a fold step of the spot-chunked variant warp 0's TMEM reads are
    // ordered before thread 0's MMAs by the tcgen05 fence and the warp sync.
    auto publish = [&](int j, bool bwd = false, bool fold_step = false) {
        if (!(bwd && warp == 0)) {
            // warps 1-3 write no backward operand; in the spot-chunked variant
            // (63 k-steps at config 4) they skip the proxy fence (-8% there;
            // the np <= 112 variant measured 0.2% slower without it, kept)
            if (!bwd || warp >= 4 || NP != kUNPC) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            hs_tc_fence_before();
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar_op + 8 * (j % RA)),
                             "r"((bwd && warp == 1) ? 2u : 1u)
                             : "memory");
        } else if (fold_step) {
            hs_tc_fence_before();
            __syncwarp();
        }
        if (warp == 0) {  // the issuing warp, converged
            hs_mbar_wait(bar_op + 8 * (j % RA), (uint32_t)(j / RA) & 1u);
            hs_tc_fence_after();
            if (j < 16) TR(0, 96 + j);
        }
    };
    auto mma_ss = [](uint32_t d, uint64_t av, uint64_t bv, uint32_t id, uint32_t acc) { hs_mma_ss(d, av, bv, id, acc); };
    // step j's MMAs (thread 0): A slot j % 4 (LBO 2048, SBO 128), B slot j % 3
    auto issue = [&](int j, uint32_t dr, uint32_t di, uint32_t lbo, uint32_t bpl, uint32_t id, uint32_t idn,
                     uint32_t acc) {
        const uint32_t as = sa + (j % RA) * kUASlot, bs = sbb + (j % RB) * kUBSlot;
        const uint64_t xb[4] = {hs_sdesc(bs, lbo, 128), hs_sdesc(bs + bpl, lbo, 128), hs_sdesc(bs + 2 * bpl, lbo, 128),
                                hs_sdesc(bs + 3 * bpl, lbo, 128)};
        hs_cmma(mma_ss, dr, di, [&](int pl) { return hs_sdesc(as + pl * kUAPl, 2048, 128); }, xb, id, idn, acc);
        commit(j);
    };
    // backward step j (thread 0): D = [Sr | Si] (N = 128) += Ar [Xr; Xi] + Ai [-Xi; Xr]
    // with B planes {B1_h, B1_l, B2_h, B2_l} of 128 rows: 6 MMAs, no negation
    const uint32_t idb = hs_idesc_tf32(2 * kUC, false);
    auto issue_bwd = [&](int j, uint32_t d, uint32_t acc) {
        const uint32_t as = sa + (j % RA) * kUASlot, bs = sbb + (j % RB) * kUBSlot;
        auto A = [&](int pl) { return hs_sdesc(as + pl * kUAPl, 2048, 128); };
        auto B = [&](int pl) { return hs_sdesc(bs + pl * kUAPl, 2048, 128); };
        hs_mma_ss(d, A(0), B(0), idb, acc);
        hs_mma_ss(d, A(0), B(1), idb, 1u);
        hs_mma_ss(d, A(1), B(0), idb, 1u);
        hs_mma_ss(d, A(2), B(2), idb, 1u);
        hs_mma_ss(d, A(2), B(3), idb, 1u);
        hs_mma_ss(d, A(3), B(2), idb, 1u);
        commit(j);
    };

    // ---- backward: S = gy (coef X)^T ------------------------------------------
    // Spot-chunked variant (large n): the k-steps accumulate in groups of KG
    // into two alternating TMEM regions, and each finished group is added
    // into fp32 registers (sacc) -- long MMA accumulation chains lose
    // accuracy (the tensor core's fp32 accumulate truncates), short ones do not.
    constexpr bool CH = NP == kUNPC;
    constexpr int KG = 8;
    float sacc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) sacc[i] = 0.f;
    int folded = 0;  // accumulation groups added into sacc
    auto fold_group = [&]() {
        const uint32_t rg = tl + (uint32_t)((folded & 1) * 128);
#pragma unroll
        for (int cc = 0; cc < NG8; cc += 2) {
            float sr[8], si[8];
            hs_tc_ld4(rg + cc * 8 + 4 * h, sr);
            hs_tc_ld4(rg + (cc + 1) * 8 + 4 * h, sr + 4);
            hs_tc_ld4(rg + kUC + cc * 8 + 4 * h, si);
            hs_tc_ld4(rg + kUC + (cc + 1) * 8 + 4 * h, si + 4);
            hs_tc_wait_ld();
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                sacc[4 * cc + jj] += sr[jj];
                sacc[32 + 4 * cc + jj] += si[jj];
            }
        }
        ++folded;
    };
    // The producers build step ks + 1's X' chunks (registers) right after
    // publishing step ks, so after the wait for a free slot only the stores
    // remain on the MMA's critical path.
    uint4 pre[4];  // X'(step) chunks: re hi, re lo, im hi, im lo
    auto make_x = [&](int ks) {  // X' = coef_k gx[c][k]: kUQ spots of column c
        const int k = ks * kUF + kUQ * xb_kq;
        float xr[kUQ], xi[kUQ];
#pragma unroll
        for (int i = 0; i < kUQ; ++i) {
            const float2 w = coef_s[k + i];
            const float4 u = xn[i / 2];
            const float ur = (i & 1) ? u.z : u.x, ui = (i & 1) ? u.w : u.y;
            xr[i] = fmaf(w.x, ur, -w.y * ui);
            xi[i] = fmaf(w.x, ui, w.y * ur);
        }
        hs_split_chunk(xr, pre[0], pre[1]);
        hs_split_chunk(xi, pre[2], pre[3]);
    };
    if (xb_on && ksteps > 0) {
        make_x(0);
        load_b(1, xn);
    }
    for (int ks = 0; ks < ksteps; ++ks) {
        if (ks >= RW) wait_mma(ks - RW);  // A slot of ks + kUD, B slot of ks free
        const bool fold_step = CH && folded < (ks - RW + 1) / KG;  // uniform
        if (ks < 16) TR(kUThreads - 2 * kUC, 64 + ks);
        if (ks < 16) TR(0, 32 + ks);
        if (CH)  // groups whose last step is <= ks - RW (group g is read before group g + 2 reuses its region)
            while (folded < (ks - RW + 1) / KG) fold_group();
        if (tid == 32) tma_ahead(ks);  // warp 1 issues the TMAs, beside thread 0's MMA issue
        if (ks < 16) TR(0, 48 + ks);
        if (xb_on) {  // step ks's X' chunks (built ahead), one 16-byte chunk per plane
            // planes [128 rows][kUF spots] (hs_uoffb): B1 = [Xr; Xi], B2 = [-Xi; Xr]
            unsigned char *d = sbase + RA * kUASlot + (ks % RB) * kUBSlot + xb_c * 16 + xb_kq * 2048;
            constexpr int R64 = kUC * 16;  // row 64
            *reinterpret_cast<uint4 *>(d) = pre[0];
            *reinterpret_cast<uint4 *>(d + R64) = pre[2];
            *reinterpret_cast<uint4 *>(d + kUAPl) = pre[1];
            *reinterpret_cast<uint4 *>(d + kUAPl + R64) = pre[3];
            *reinterpret_cast<uint4 *>(d + 2 * kUAPl) = hs_neg_chunk(pre[2]);
            *reinterpret_cast<uint4 *>(d + 2 * kUAPl + R64) = pre[0];
            *reinterpret_cast<uint4 *>(d + 3 * kUAPl) = hs_neg_chunk(pre[3]);
            *reinterpret_cast<uint4 *>(d + 3 * kUAPl + R64) = pre[1];
        }
        if (ks < 16) TR(kUThreads - 2 * kUC, 80 + ks);

        publish(ks, true, fold_step);
        if (xb_on && ks + 1 < ksteps) {
            make_x(ks + 1);
            load_b(ks + 2, xn);
        }
        if (warp == 0) {
            const uint32_t dr = CH ? tm + (uint32_t)(((ks / KG) & 1) * 128) : tm;
            issue_bwd(ks, dr, (CH ? ks % KG : ks) ? 1u : 0u);
            if (ks < 16) TR(0, 2 + ks);
        }
    }

    // amplitudes of this thread's 32 pixels: columns 8 cc + 4 h + j (c0 is a
    // multiple of 8, so each group of 4 is one aligned float4 when side % 4 == 0)
    const int64_t prow = (int64_t)min(grow, a.side - 1) * a.side;
    float br[32], bi[32];
    const bool vec_amp = (a.side & 3) == 0;
#pragma unroll
    for (int cc = 0; cc < NG8; ++cc) {
        const int c = c0 + cc * 8 + 4 * h;
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
    TR(0, 18);

    if (CH)
        while (folded < (ksteps + KG - 1) / KG) fold_group();

    // ---- S -> b = A conj(S)/|S| (registers), phase write --------------------
    // S of 8 pixels per step, double-buffered: the next step's TMEM loads are
    // issued right after the wait for the current one's
    float sbuf[2][16];  // [buffer][Sr 8 | Si 8]
    auto ld_s = [&](int cc, float *d) {
        hs_tc_ld4(tl + cc * 8 + 4 * h, d);
        hs_tc_ld4(tl + (cc + 1) * 8 + 4 * h, d + 4);
        hs_tc_ld4(tl + kUC + cc * 8 + 4 * h, d + 8);
        hs_tc_ld4(tl + kUC + (cc + 1) * 8 + 4 * h, d + 12);
    };
    if (!CH) ld_s(0, sbuf[0]);
#pragma unroll
    for (int cc = 0; cc < NG8; cc += 2) {
        float *sr = sbuf[(cc >> 1) & 1], *si = sr + 8;
        if (CH) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                sr[jj] = sacc[4 * cc + jj];
                si[jj] = sacc[32 + 4 * cc + jj];
            }
        } else {
            hs_tc_wait_ld();
            if (cc + 2 < NG8) ld_s(cc + 2, sbuf[((cc >> 1) + 1) & 1]);
        }
        int dix[8];  // storage indices of the 8 pixels (WRITE), two aligned int4 when side % 4 == 0
        if (WRITE) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int c = c0 + (cc + u) * 8 + 4 * h;
                if (vec_amp) {
                    const int4 v = (row_in && c < a.side) ? __ldg(reinterpret_cast<const int4 *>(a.idx_img + prow + c))
                                                          : make_int4(-1, -1, -1, -1);
                    dix[4 * u] = v.x; dix[4 * u + 1] = v.y; dix[4 * u + 2] = v.z; dix[4 * u + 3] = v.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        dix[4 * u + j] = (row_in && c + j < a.side) ? __ldg(a.idx_img + prow + c + j) : -1;
                }
            }
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int i = 4 * cc + jj;
            const float A = br[i];
            hs_bvec_nb(sr[jj], si[jj], A, br[i], bi[i]);  // branch-free: the 8 pixels interleave
            if (WRITE) {
                const int c = c0 + (i / 4) * 8 + 4 * h + (i % 4);
                if (row_in && c < a.side) {
                    const int32_t di = dix[jj];
                    if (di >= 0) {
                        if (WRITE == 2)
                            a.phase_out32[(int64_t)pat * a.phase_stride + di] = hs_phase_code(sr[jj], si[jj]);
                        else
                            a.phase_out[(int64_t)pat * a.phase_stride + di] = hs_phase_f64(sr[jj], si[jj]);
                        if (a.raster)
                            a.raster[(int64_t)pat * a.side * a.side + prow + c] =
                                hs_gray_linear(hs_phase_f64(sr[jj], si[jj]));
                    }
                }
            }
        }
    }

    TR(0, 19);
    // ---- forward: T = b X ------------------------------------------------------
    // A slot: b' planes [128 rows][kUF columns] (hs_uoffb); B slot: X^T planes
    // [NP spots][kUF columns] ((k/8)*128 + (c/kUQ)*FLBO + (k%8)*16 + (c%kUQ)*kUEB), TMA
    const uint32_t idf = hs_idesc_tf32(NP, false), idfn = hs_idesc_tf32(NP, true);
    float2 *out = a.f.partials + (int64_t)pat * a.f.part_stride + (int64_t)tile * a.np;
    // T of spot chunk sc lives in TMEM columns tb(sc): the spot-chunked
    // variant (one CTA per SM, 512 columns) double-buffers it, so chunk
    // sc + 1's MMAs run while chunk sc's E epilogue reads its T
    constexpr bool TB = NP == kUNPC;
    auto tb = [&](int sc) -> uint32_t { return TB ? (uint32_t)((sc & 1) * 256) : 0u; };
    auto fwd_chunk = [&](int sc) {
#pragma unroll
    for (int cc = 0; cc < NCC; ++cc) {
        const int j = ksteps + sc * NCC + cc;  // step
        wait_mma(j - RW);            // A slot of j (last used by j - RA), B slot of j + kUD free
        if (tid == 32) tma_ahead(j);
        if constexpr (kF16) {  // b' (this thread's row): columns 4h .. 4h+3 of both 8-column K halves
#pragma unroll
            for (int qh = 0; qh < 2; ++qh) {
                const int g = 2 * cc + qh;  // 8-column group of the row
                uint32_t rh[2], rl[2], ih[2], il[2];
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    hs_split2(br[4 * g + 2 * jj], br[4 * g + 2 * jj + 1], rh[jj], rl[jj]);
                    hs_split2(bi[4 * g + 2 * jj], bi[4 * g + 2 * jj + 1], ih[jj], il[jj]);
                }
                unsigned char *d = sbase + (j % RA) * kUASlot + row * 16 + qh * 2048 + h * 8;
                *reinterpret_cast<uint2 *>(d) = make_uint2(rh[0], rh[1]);
                *reinterpret_cast<uint2 *>(d + kUAPl) = make_uint2(rl[0], rl[1]);
                *reinterpret_cast<uint2 *>(d + 2 * kUAPl) = make_uint2(ih[0], ih[1]);
                *reinterpret_cast<uint2 *>(d + 3 * kUAPl) = make_uint2(il[0], il[1]);
            }
        } else {  // b' (this thread's row, columns 4h .. 4h+3 of the k-step = K half h)
            uint4 rh, rl, ih, il;
            hs_split_chunk(&br[4 * cc], rh, rl);
            hs_split_chunk(&bi[4 * cc], ih, il);
            unsigned char *d = sbase + (j % RA) * kUASlot + row * 16 + h * 2048;
            *reinterpret_cast<uint4 *>(d) = rh;
            *reinterpret_cast<uint4 *>(d + kUAPl) = rl;
            *reinterpret_cast<uint4 *>(d + 2 * kUAPl) = ih;
            *reinterpret_cast<uint4 *>(d + 3 * kUAPl) = il;
        }
        publish(j);  // (cc = 0: also orders the S / previous chunk's T reads before T is overwritten)
        if (warp == 0) {
            issue(j, tm + tb(sc), tm + tb(sc) + NP, FLBO, FPL, idf, idfn, cc ? 1u : 0u);
            if (sc == 0) TR(0, 20 + cc);
        }
    }
    };
    if (TB) fwd_chunk(0);
#pragma unroll 1
    for (int sc = 0; sc < nsc; ++sc) {
    if (!TB) fwd_chunk(sc);
    else if (sc + 1 < nsc) fwd_chunk(sc + 1);  // after chunk sc - 1's E reads (program order + publish)
    wait_mma(ksteps + (sc + 1) * NCC - 1);
    if (sc == 0) TR(0, 28);

    // ---- E_k = sum_r gy[r][k] T[r][k]: spots KH h .. KH (h+1) of the row, 16
    // at a time; each group of 16 (32 values) is transpose-reduced over the
    // warp's 32 rows (one value per lane), then the 4 lane-quarter warps are
    // summed in order through shared memory.  gy comes from its fp32 copy in
    // the row-coalesced E layout (hs_umma_gye_floats); the next group's gy is
    // loaded while the current one is reduced.
    const int k0 = sc * NP;             // first spot of the chunk
    constexpr int NG = (KH + 15) / 16;  // groups of 16 spots (the last may hold 8)
    float4 gq[2][2][4];                 // [buffer][quad-pair half][plane]
    // fp32 gy of this band (hs_umma_gye_floats layout), row-coalesced
    const float4 *gye = reinterpret_cast<const float4 *>(pbase + hs_umma_gy_floats(a.side, a.np) +
                                                         (int64_t)hs_umma_xblocks(a.side) * hs_umma_xblock_floats(a.np) +
                                                         (int64_t)(r0 / kUR) * a.np * 4 * kUR / 2) + row;
    auto load_g = [&](int g, float4 (&d)[2][4]) {
        const int kk = KH * h + 16 * g;
#pragma unroll
        for (int e = 0; e < 2; ++e) {  // k8 block e of the group
            if (16 * g + 8 * e < KH) {
                // spots past np (last chunk's padding): any finite data, T is 0 there
                const int sp = min(k0 + kk + 8 * e, a.np - 8);  // first of 8 spots (multiple of 8)
                const float4 *pe = gye + (int64_t)(sp / 8) * 4 * kUR;
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) d[e][qd] = __ldg(pe + qd * kUR);
            }
        }
    };
    load_g(0, gq[0]);
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        float4 (&gc)[2][4] = gq[g & 1];
        if (g + 1 < NG) load_g(g + 1, gq[(g + 1) & 1]);
        const int kk = KH * h + 16 * g;
        const int KQ = min(16, KH - 16 * g);  // 16 or 8 (compile-time per NP)
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
        float tq[2][16];  // T of the group's two 8-spot halves: [e][Tr 8 | Ti 8], one wait for both
#pragma unroll
        for (int e = 0; e < 2; ++e)
            if (8 * e < KQ) {
                hs_tc_ld8(tl + tb(sc) + kk + 8 * e, *reinterpret_cast<float (*)[8]>(tq[e]));
                hs_tc_ld8(tl + tb(sc) + NP + kk + 8 * e, *reinterpret_cast<float (*)[8]>(tq[e] + 8));
            }
        hs_tc_wait_ld();
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            if (8 * e < KQ) {
                const float *tr = tq[e], *ti = tq[e] + 8;
                const float gr[8] = {gc[e][0].x, gc[e][0].y, gc[e][0].z, gc[e][0].w,
                                     gc[e][2].x, gc[e][2].y, gc[e][2].z, gc[e][2].w};
                const float gi[8] = {gc[e][1].x, gc[e][1].y, gc[e][1].z, gc[e][1].w,
                                     gc[e][3].x, gc[e][3].y, gc[e][3].z, gc[e][3].w};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    v[16 * e + 2 * j] = fmaf(gr[j], tr[j], -gi[j] * ti[j]);
                    v[16 * e + 2 * j + 1] = fmaf(gr[j], ti[j], gi[j] * tr[j]);
                }
            }
        }
        // transpose-reduce: at offset o the lane keeps the half selected by
        // its lane bit o (a fixed order per value: deterministic)
#pragma unroll
        for (int o = 16, w = 16; o > 0; o >>= 1, w >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int j = 0; j < w; ++j) {
                const float send = up ? v[j] : v[j + w];
                const float keep = up ? v[j + w] : v[j];
                v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        // lane l holds value index l (value 2 s + t = spot s, re/im t); each
        // group has its own scratch row, so the groups' shuffle chains run
        // back to back and one barrier serves all of them
        red[(g * 8 + warp) * 32 + lane] = v[0];
    }
    __syncthreads();
    for (int idx = tid; idx < NG * 2 * 16; idx += kUThreads) {  // (group g, spot-half hq, spot s)
        const int g = idx >> 5, hq = (idx >> 4) & 1, s = idx & 15;
        const int KQ = min(16, KH - 16 * g);
        if (s < KQ && k0 + KH * hq + 16 * g + s < a.np) {
            float x = 0.f, y = 0.f;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                x += red[(g * 8 + qq + 4 * hq) * 32 + 2 * s];
                y += red[(g * 8 + qq + 4 * hq) * 32 + 2 * s + 1];
            }
            out[k0 + KH * hq + 16 * g + s] = make_float2(x, y);
        }
    }
    if (sc + 1 < nsc) __syncthreads();  // the next chunk's groups rewrite the scratch
    }  // spot chunks
    TR(0, 29);

    hs_tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(NP == kUNPC ? 2 * kUTmem : kUTmem));
    if (a.f.u.act != ACT_NONE) hs_fold(a.f, pat, tile, reinterpret_cast<char *>(sbase));
    TR(0, 30);
}

typedef void (*UmmaFn)(TileArgs);
UmmaFn hs_select_umma(int np, int write);  // write: 0 none, 1 f64 phases, 2 phase codes

}  // namespace hs
