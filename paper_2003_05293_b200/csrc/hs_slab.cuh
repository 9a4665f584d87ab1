// hs_slab.cuh -- compressed-window fused pass with the gx table staged in
// shared memory (solver iterations 1..I-2, solvers.py:212-230).
//
// A window is a random 1/16 of the aperture (a storage-order range of the
// seeded permutation, optics.py:184-187), so the gx row a pixel needs is a
// random row of the pattern's table.  Gathering those rows from L2 left the
// window pass latency-bound (hs_win.cuh).  Here the grid is cut into column
// slabs of `sw` columns whose gx rows fit in shared memory (sw * np * 8 B,
// ~180 KB); the window list is ordered (slab, row-run) and cut into chunks of
// 32 streams x kSlabP entries that never cross a slab.  A CTA
//
//   * stages its slab's gx rows with TMA bulk copies (cp.async.bulk onto an
//     mbarrier carrying the byte count) -- re-staged only when its next chunk
//     lies in another slab;
//   * runs 32 pixel streams: G lanes per pixel (G = 8: 4 streams per warp,
//     8 warps; G = 16: 2 per warp, 16 warps), lane g owning spots
//     VEC (g + G j) + h (VEC = 16 / G complex per shared load, so every group
//     load is one conflict-free 128-B wavefront);
//   * takes two pixels of a row-run per trip: their backward partials are
//     finished by a transpose-reduce (half the group finishes each pixel),
//     b = A conj(S)/|S| is exchanged by one shuffle, and both feed the
//     forward accumulators T = sum_p b_p gx[c_p] of the run;
//   * keeps V = coef gy[row] and T per run in registers (the streams of a
//     warp change row on the same trip: runs are sorted by length and
//     grouped per warp), flushing E += gy[row] T into per-stream shared
//     memory at run ends.
//
// Complex MACs are FFMA2 (hs_f2.cuh).  Per pixel-spot pair: one 8-B shared
// read + two complex MACs (backward kernels.py:99-119, forward
// kernels.py:122-144).  A chunk's partial is its 32 streams' E summed in a
// fixed order; chunks are folded by hs_fold -- the reduction shape depends
// only on the list, so results are bitwise independent of the batch size
// and of how many chunks a CTA streams.
#pragma once

#include "hs_f2.cuh"
#include "hs_kernels.cuh"

namespace hs {

#ifndef HS_SLAB_L1PF
#define HS_SLAB_L1PF 0  // 1: whole-chunk CTAs prefetch the next run's gy row into L1 (measured neutral)
#endif
constexpr int kSlabG = 16;                       // lanes per pixel (8 or 16)
constexpr int kSlabThreads = 32 * kSlabG;        // 32 streams of kSlabG lanes
constexpr int kSlabWarps = kSlabThreads / 32;
constexpr int kSlabStreams = 32;                 // pixel streams per CTA
constexpr int kSlabP = 32;                       // entries per stream per chunk
constexpr int kSlabL = kSlabStreams * kSlabP;    // entries per chunk
// Entries in shared memory: [2 chunks][32 streams][kSlabP]; odd streams
// store entry t at t ^ 2, so the two streams of a warp read their entry
// pairs (t, t+1) from different banks (one wavefront per warp instead of two)
constexpr int kEntStride = kSlabP;
constexpr int kEntBuf = kSlabStreams * kEntStride;  // one chunk's entries in smem
__host__ __device__ constexpr int hs_ent_swz(int stream) { return (stream & 1) << 1; }
constexpr int kSlabSmemBudget = 220 * 1024;      // dynamic smem cap per CTA
constexpr int kBulkPiece = 32 * 1024;            // bytes per cp.async.bulk

struct SlabArgs {
    const int2 *ent;          // (rc, amp bits) per entry, chunk-major, padded to kSlabL
    const int32_t *chunk_c0;  // first grid column of each chunk's slab
    int32_t sw;               // slab width (columns)
    int32_t side;
    int32_t cpc;              // chunks per CTA (divides kGroup)
    int64_t tab_stride;       // side * np
    const float2 *gx, *gy;    // [B][side][np]
    const float2 *coef;       // [B][np]
    FoldArgs f;
    unsigned long long *trace;  // timing probe of one CTA (HS_SLAB_TRACE), normally null
};

__host__ __device__ constexpr size_t hs_slab_fixed_bytes(int np)
{
    // per-stream E [32][np] float2 + entries [2][32][kEntStride] int2 + coef [np] float2
    return (size_t)kSlabStreams * np * 8 + (size_t)2 * kEntBuf * 8 + (size_t)np * 8;
}

// Widest slab whose gx rows fit next to the per-CTA scratch.
__host__ __device__ constexpr int hs_slab_width(int np, int side)
{
    return ((int)((kSlabSmemBudget - hs_slab_fixed_bytes(np)) / (sizeof(float2) * np)) & ~7) < side
               ? ((int)((kSlabSmemBudget - hs_slab_fixed_bytes(np)) / (sizeof(float2) * np)) & ~7)
               : side;
}

__host__ __device__ constexpr size_t hs_slab_smem_bytes(int np, int sw)
{
    return sizeof(float2) * (size_t)np * sw + hs_slab_fixed_bytes(np);
}

__device__ __forceinline__ float2 hs_lds2(uint32_t addr)
{
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

// PIPE = false: pair trips (two pixels of a run per trip, transpose-reduce
// across the two halves of the lane group).  PIPE = true: one pixel per step,
// software-pipelined -- the butterfly of pixel t runs while the backward of
// pixel t+1 issues (both in one basic block, so ptxas interleaves the
// shuffle latency with FFMA2 work); see the main loop below.
template <int NS, int G, bool HALF, bool PIPE = false>
__global__ void __launch_bounds__(HALF ? 16 * G : 32 * G, 1) hs_slab_kernel(const SlabArgs a)
{
    constexpr int WPC = G;              // warps of a whole chunk (32 streams)
    constexpr int NW = HALF ? WPC / 2 : WPC;  // warps in this CTA
    constexpr int NT = 32 * NW;         // threads
    constexpr int GPW = 32 / G;         // pixel groups (streams) per warp
    constexpr int VEC = 16 / G;         // complex values per lane per shared load
    constexpr int NP = 16 * NS;
    constexpr int SPL = VEC * NS;       // spots per lane
    constexpr int P = kSlabP;
    static_assert(GPW * WPC == kSlabStreams, "32 streams per chunk");
    extern __shared__ float4 sm4[];
    __shared__ __align__(8) unsigned long long bar;

    hs_pdl_launch_next();
    const bool trc = a.trace && blockIdx.x == (gridDim.x > 20 ? 20u : gridDim.x / 2) && blockIdx.y == 0;
    auto TR = [&](int slot) {
#if HS_PROBES
        if (trc && threadIdx.x == 0) a.trace[slot] = clock64();
#else
        (void)trc, (void)slot;
#endif
    };
    TR(0);
    const int pat = blockIdx.y;
    // fold units are half-chunks (16 streams); a whole-chunk CTA streams cpc
    // chunks, a half-chunk CTA (small batches: twice the CTAs) one half
    const int half = HALF ? (int)(blockIdx.x & 1) : 0;
    const int q0 = a.f.chunk_base / 2 + (HALF ? (int)(blockIdx.x >> 1) : (int)blockIdx.x * a.cpc);
    const int nq = HALF ? 1 : min(a.cpc, a.f.chunk_end / 2 - q0);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int gw = warp + half * NW;    // warp index in the chunk layout
    const int g = lane & (G - 1), s = lane / G;
    const bool lo = g < G / 2;
    const int stream = gw * GPW + s;

    float2 *Xs = reinterpret_cast<float2 *>(sm4);                 // [sw][NP]
    float2 *Es = Xs + (size_t)a.sw * NP;                            // [32][NP]
    int2 *Ent = reinterpret_cast<int2 *>(Es + kSlabStreams * NP);   // [2][32][kEntStride]
    float2 *coef_s = reinterpret_cast<float2 *>(Ent + 2 * kEntBuf); // [NP]
    // lane's first complex in a table row: spot VEC g (stride VEC G per j)
    const uint32_t xs_a = hs_smem_addr(Xs) + 8u * VEC * g;
    const uint32_t es_a = hs_smem_addr(Es) + 8u * (stream * NP + VEC * g);
    const uint32_t ent_a = hs_smem_addr(Ent);
    const uint32_t cf_a = hs_smem_addr(coef_s) + 8u * VEC * g;

    for (int k = tid; k < kSlabStreams * NP; k += NT) Es[k] = make_float2(0.f, 0.f);

    // per-warp entry staging: the warp's GPW streams of chunk q are the
    // GPW * P entries [w GPW P, (w+1) GPW P) of the chunk
    constexpr int EPL = GPW * P / 32;  // entries per lane
    int2 ent_reg[EPL];
    auto fetch_ent = [&](int qi) {
        if (qi < nq)
#pragma unroll
            for (int k = 0; k < EPL; ++k)
                ent_reg[k] = __ldg(a.ent + (int64_t)(q0 + qi) * kSlabL + gw * GPW * P + lane + 32 * k);
    };
    auto store_ent = [&](int qi) {
        if (qi < nq)
#pragma unroll
            for (int k = 0; k < EPL; ++k) {
                const int i = lane + 32 * k;  // entry i of the warp's GPW streams
                const int st = gw * GPW + i / P;
                Ent[(qi & 1) * kEntBuf + st * kEntStride + ((i % P) ^ hs_ent_swz(st))] = ent_reg[k];
            }
    };
    fetch_ent(0);
    store_ent(0);
    fetch_ent(1);
    store_ent(1);
    const uint32_t bar_a = hs_smem_addr(&bar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const float2 *__restrict__ gx = a.gx + (int64_t)pat * a.tab_stride;
    const float2 *__restrict__ Yrow0 = a.gy + (int64_t)pat * a.tab_stride;
    const float2 *__restrict__ Y = Yrow0 + VEC * g;
    uint32_t phase = 0;
    int c0 = -1;

    // Stage the gx rows of slab [cs, cs + sw) (all threads call; one issues).
    auto stage = [&](int cs) {
        __syncthreads();  // previous readers of Xs are done
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int ncol = min(a.sw, a.side - cs);
            const uint32_t bytes = (uint32_t)ncol * NP * 8u;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(bytes)
                         : "memory");
            const char *src = reinterpret_cast<const char *>(gx + (int64_t)cs * NP);
            const uint32_t dst = hs_smem_addr(Xs);
            for (uint32_t off = 0; off < bytes; off += kBulkPiece) {
                const uint32_t len = min((uint32_t)kBulkPiece, bytes - off);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        dst + off),
                    "l"(src + off), "r"(len), "r"(bar_a)
                    : "memory");
            }
        }
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                : "=r"(done)
                : "r"(bar_a), "r"(phase)
                : "memory");
        }
        phase ^= 1u;
        c0 = cs;
    };

    // lane state (SPL spots): V = coef * gy[row], gy[row], T packed (re, im)
    float vr[SPL], vi[SPL], yr_[SPL], yi_[SPL];
    f2x tt[SPL];
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
        vr[k] = vi[k] = yr_[k] = yi_[k] = 0.f;
        tt[k] = 0ull;
    }

    // shared loads of VEC complex values (one lane's slice of a row)
    auto lds_vec = [&](uint32_t addr, f2x *d) {
        if constexpr (VEC == 2)
            asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(d[0]), "=l"(d[VEC - 1]) : "r"(addr));
        else
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(d[0]) : "r"(addr));
    };
    auto sts_vec = [&](uint32_t addr, const f2x *d) {
        if constexpr (VEC == 2)
            asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(addr), "l"(d[0]), "l"(d[VEC - 1]) : "memory");
        else
            asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(d[0]) : "memory");
    };
    auto load_x = [&](int rc, f2x (&x)[SPL]) {
        const uint32_t row = xs_a + 8u * NP * (uint32_t)(rc & 0xffff);  // slab-local column
#pragma unroll
        for (int j = 0; j < NS; ++j) lds_vec(row + 8u * VEC * G * j, &x[VEC * j]);
    };
    auto flush = [&]() {  // Es[stream] += Y * T ; T = 0
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            f2x e[VEC];
            lds_vec(es_a + 8u * VEC * G * j, e);
#pragma unroll
            for (int h = 0; h < VEC; ++h) {
                const int k = VEC * j + h;
                f2_cmac1(e[h], yr_[k], yi_[k], tt[k]);
                tt[k] = 0ull;
            }
            sts_vec(es_a + 8u * VEC * G * j, e);
        }
    };
    // Half-chunk CTAs (small batches: 8 warps per SM, where the gy-row load
    // latency at each run start is exposed, ncu long_sb) keep the next run's
    // gy row in registers (gyn, row rnext), loaded a whole run ahead from the
    // row hint in the list; whole-chunk CTAs have no registers to spare.
    constexpr bool PREF = HALF;
    float2 gyn[PREF ? SPL : 1];
    int rnext = -1;
    auto load_next = [&](int r) {
        if constexpr (PREF) {
            const float2 *yrow = Y + (int64_t)r * NP;
#pragma unroll
            for (int j = 0; j < NS; ++j)
#pragma unroll
                for (int h = 0; h < VEC; ++h) gyn[VEC * j + h] = __ldg(yrow + VEC * G * j + h);
            rnext = r;
        }
    };
    auto new_row = [&](int r) {  // Y = gy[r], V = coef * Y
        const float2 *yrow = Y + (int64_t)r * NP;
        const bool pre = PREF && rnext == r;
#pragma unroll
        for (int j = 0; j < NS; ++j) {
#pragma unroll
            for (int h = 0; h < VEC; ++h) {
                const int k = VEC * j + h;
                const float2 q = pre ? gyn[PREF ? k : 0] : __ldg(yrow + VEC * G * j + h);
                const float2 w = hs_lds2(cf_a + 8u * (VEC * G * j + h));
                yr_[k] = q.x;
                yi_[k] = q.y;
                vr[k] = fmaf(w.x, q.x, -w.y * q.y);
                vi[k] = fmaf(w.x, q.y, w.y * q.x);
            }
        }
    };

    __syncwarp();
    stage(__ldg(a.chunk_c0 + q0));  // gx (tables) and lists: inputs of the whole solve
    // -- everything below reads the previous pass's results (status, coef)
    hs_pdl_wait_prev();
    // coefficient and status loads in flight together (one L2 round trip on
    // the pass's critical path, which is what a single hologram waits on)
    static_assert(NP <= NT, "one coefficient per thread");
    const float2 cfv = tid < NP ? a.coef[(int64_t)pat * NP + tid] : make_float2(0.f, 0.f);
    if (a.f.u.status[pat] != 0) return;  // uniform per CTA
    if (tid < NP) coef_s[tid] = cfv;
    __syncthreads();
    int rcur = -1;
    // smem address of this stream's entries in chunk buffer 0 / 1
    const uint32_t ent0 = ent_a + 8u * (stream * kEntStride), ent1 = ent0 + 8u * kEntBuf;
    const uint32_t eswz = 8u * hs_ent_swz(stream);  // byte offset XOR of entry pairs
    int4 en;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(en.x), "=r"(en.y), "=r"(en.z), "=r"(en.w) : "r"(ent0 + eswz));

    // One pair-trip = two pixels per group (entries t, t+1 of a run; runs are
    // padded to even length, so both share the row).  Lanes g < G/2 finish
    // pixel t ("mine") and hand t+1's partial over, lanes g >= G/2 the
    // reverse, so the transpose-reduce needs no selects.
    auto pair = [&](int qi, int t) {
        const int4 e = en;
        const int rc_m = lo ? e.x : e.z, rc_o = lo ? e.z : e.x;
        const float A_m = __int_as_float(lo ? e.y : e.w);
        f2x xm[SPL], xo[SPL];
        load_x(rc_m, xm);
        load_x(rc_o, xo);
        {   // next pair's entries (the next chunk's buffer after the last pair;
            // past the CTA's last chunk the read is stale and unused)
            const uint32_t nxt = ((t + 2 < P) ? ((qi & 1) ? ent1 : ent0) + (8u * (t + 2) ^ eswz)
                                              : ((qi & 1) ? ent0 : ent1) + eswz);
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(en.x), "=r"(en.y), "=r"(en.z), "=r"(en.w)
                         : "r"(nxt));
        }
        const int r = e.x >> 16;
        if (r != rcur) {  // warp-uniform: a warp's runs change row together
            if (rcur >= 0) flush();
            new_row(r);
            rcur = r;
            // the second entry's row bits carry the row of this stream's next
            // run: load it a run ahead of new_row (PREF), else pull it into L1
            const int rn = e.z >> 16;
            if constexpr (PREF) {
                if (rn != r) load_next(rn);
            } else if (HS_SLAB_L1PF && rn != r && g < NS + 1) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(Yrow0 + (int64_t)rn * NP + min(16 * g, NP - 1)));
            }
        }
        // backward partials of both pixels over this lane's spots (FFMA2)
        f2x m0 = 0ull, m1 = 0ull, o0 = 0ull, o1 = 0ull;
#pragma unroll
        for (int k = 0; k < SPL; ++k) {
            f2_cmac1((k & 1) ? m1 : m0, vr[k], vi[k], xm[k]);
            f2_cmac1((k & 1) ? o1 : o0, vr[k], vi[k], xo[k]);
        }
        float kr = f2_lo(m0) + f2_lo(m1), ki = f2_hi(m0) + f2_hi(m1);
        const float sr_o = f2_lo(o0) + f2_lo(o1), si_o = f2_hi(o0) + f2_hi(o1);
        // transpose-reduce over the G lanes (commutative butterflies: every
        // lane of a half ends with identical bits)
        kr += __shfl_xor_sync(0xffffffffu, sr_o, G / 2);
        ki += __shfl_xor_sync(0xffffffffu, si_o, G / 2);
#pragma unroll
        for (int o = G / 4; o > 0; o >>= 1) {
            kr += __shfl_xor_sync(0xffffffffu, kr, o);
            ki += __shfl_xor_sync(0xffffffffu, ki, o);
        }
        float mr, mi;
        hs_bvec_nb(kr, ki, A_m, mr, mi);
        const float orr = __shfl_xor_sync(0xffffffffu, mr, G / 2);
        const float oi = __shfl_xor_sync(0xffffffffu, mi, G / 2);
#pragma unroll
        for (int k = 0; k < SPL; ++k) f2_cmac1(tt[k], mr, mi, xm[k]);
#pragma unroll
        for (int k = 0; k < SPL; ++k) f2_cmac1(tt[k], orr, oi, xo[k]);
    };

    // End of chunk qi: flush, sum the 32 streams in a fixed order, reset, stage.
    auto chunk_end = [&](int qi, int cs_next) {
        if (rcur >= 0) flush();
        rcur = -1;
        // the warp's GPW streams: symmetric butterfly adds, kept in stream
        // GPW gw's row; then each half's 8 warp rows summed in warp order
        {
            const uint32_t w0 = hs_smem_addr(Es) + 8u * (GPW * gw * NP + VEC * g);
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                f2x v[VEC];
                lds_vec(es_a + 8u * VEC * G * j, v);
#pragma unroll
                for (int h = 0; h < VEC; ++h) {
                    float x = f2_lo(v[h]), y = f2_hi(v[h]);
#pragma unroll
                    for (int o = G; o < 32; o <<= 1) {
                        x += __shfl_xor_sync(0xffffffffu, x, o);
                        y += __shfl_xor_sync(0xffffffffu, y, o);
                    }
                    v[h] = f2_pack(x, y);
                }
                if (s == 0) {
                    sts_vec(w0 + 8u * VEC * G * j, v);
                } else {
                    const f2x z[VEC == 2 ? 2 : 1] = {};
                    sts_vec(es_a + 8u * VEC * G * j, z);
                }
            }
        }
        // whole-chunk CTAs: each half-chunk's 8 warps sync on their own named
        // barrier (1 + half), so one half's reduction does not wait for the
        // other half's last trip
        constexpr int HALVES = HALF ? 1 : 2;
        const int my_half = HALF ? half : gw / (WPC / 2);
        if constexpr (HALF) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + my_half), "n"(NT / 2) : "memory");
        for (int idx = HALF ? tid : tid - my_half * (NT / 2); idx < NP; idx += HALF ? NT : NT / 2) {
            const int hh = my_half, k = idx;
            float x = 0.f, y = 0.f;
#pragma unroll
            for (int w = 0; w < WPC / 2; ++w) {
                const int row = GPW * (hh * (WPC / 2) + w) * NP + k;
                const float2 v = Es[row];
                x += v.x;
                y += v.y;
                Es[row] = make_float2(0.f, 0.f);
            }
            a.f.partials[(int64_t)pat * a.f.part_stride + (int64_t)(2 * (q0 + qi) + hh) * NP + k] =
                make_float2(x, y);
        }
        store_ent(qi + 2);  // chunk qi's buffer is consumed
        __syncwarp();
        if (qi + 1 < nq) {
            const int cs = cs_next;  // loaded at the chunk's start (a register: the halves do not sync here)
            if (cs != c0)
                stage(cs);        // begins with __syncthreads
            else if constexpr (HALF)
                __syncthreads();  // Es reset visible before the next flushes
            else
                asm volatile("bar.sync %0, %1;" ::"r"(1 + my_half), "n"(NT / 2) : "memory");
        }
    };

    // ---- pipelined per-pixel steps (PIPE) ----
    // backward partial of one pixel over this lane's spots (two FFMA2 chains)
    auto bwd = [&](const f2x (&x)[SPL], float &sr, float &si) {
        f2x m0 = 0ull, m1 = 0ull;
#pragma unroll
        for (int k = 0; k < SPL; ++k) f2_cmac1((k & 1) ? m1 : m0, vr[k], vi[k], x[k]);
        sr = f2_lo(m0) + f2_lo(m1);
        si = f2_hi(m0) + f2_hi(m1);
    };
    // sum over the G lanes, transposed over (re, im): after the first
    // exchange the low half of the group carries Re, the high half Im, so
    // one value per lane goes through the remaining levels (commutative
    // butterflies: every lane of a half ends with identical bits)
    auto chain = [&](float sr, float si) {
        float keep = lo ? sr : si;
        keep += __shfl_xor_sync(0xffffffffu, lo ? si : sr, G / 2);
#pragma unroll
        for (int o = G / 4; o > 0; o >>= 1) keep += __shfl_xor_sync(0xffffffffu, keep, o);
        return keep;
    };
    auto bfin = [&](float keep, float A, float &br, float &bi) {
        const float other = __shfl_xor_sync(0xffffffffu, keep, G / 2);
        hs_bvec_nb(lo ? keep : other, lo ? other : keep, A, br, bi);
    };
    auto fwd = [&](const f2x (&x)[SPL], float br, float bi) {
#pragma unroll
        for (int k = 0; k < SPL; ++k) f2_cmac1(tt[k], br, bi, x[k]);
    };
    // One chunk: entries (t, t+1) of a stream always lie in one run (runs are
    // padded to even length and the two runs of a warp to the same length),
    // so the row can only change at even t, warp-uniformly.  Per step the
    // reduction of the previous pixel and the backward of the next one form
    // one branch-free block; a row change re-runs the (already loaded)
    // pixel's backward with the new V after the flush.
    auto pipe_chunk = [&](uint32_t eb) {
        int4 e;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w) : "r"(eb + eswz));
        rcur = e.x >> 16;
        new_row(rcur);
        f2x xa[SPL], xb[SPL];
        float sr, si, A = __int_as_float(e.y);
        load_x(e.x, xa);
        bwd(xa, sr, si);
#pragma unroll 1
        for (int t = 0; t < P; t += 2) {
            // pixel t (xa, partials sr/si) -> forward; pixel t+1 (same run) -> backward
            load_x(e.z, xb);
            const float A1 = __int_as_float(e.w);
            float s1r, s1i, br, bi;
            {
                const float keep = chain(sr, si);
                bwd(xb, s1r, s1i);
                bfin(keep, A, br, bi);
            }
            fwd(xa, br, bi);
            if (t + 2 < P) {
                asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w)
                             : "r"(eb + (8u * (t + 2) ^ eswz)));
                load_x(e.x, xa);
                A = __int_as_float(e.y);
                const float keep = chain(s1r, s1i);
                bwd(xa, sr, si);
                bfin(keep, A1, br, bi);
                fwd(xb, br, bi);
                const int r = e.x >> 16;
                if (r != rcur) {  // warp-uniform
                    flush();
                    new_row(r);
                    rcur = r;
                    bwd(xa, sr, si);
                }
            } else {
                bfin(chain(s1r, s1i), A1, br, bi);
                fwd(xb, br, bi);
            }
        }
    };

    TR(1);
    for (int qi = 0; qi < nq; ++qi) {
        if (qi < 16) TR(2 + 3 * qi);
        fetch_ent(qi + 2);
        // the next chunk's slab origin, loaded now, used at the chunk's end
        const int cs_next = (qi + 1 < nq) ? __ldg(a.chunk_c0 + q0 + qi + 1) : 0;
        if constexpr (PIPE) {
            pipe_chunk((qi & 1) ? ent1 : ent0);
        } else {
#pragma unroll 1
            for (int t = 0; t < P; t += 16) {
#pragma unroll
                for (int u = 0; u < 16; u += 2) pair(qi, t + u);
            }
        }
        if (qi < 16) TR(3 + 3 * qi);
        chunk_end(qi, cs_next);
        if (qi < 16) TR(4 + 3 * qi);
    }
    TR(60);
    if (a.f.u.act != ACT_NONE) {
        __syncthreads();
        hs_fold(a.f, pat, 2 * q0 + half, reinterpret_cast<char *>(Es), HALF ? 1 : 2 * nq);
    }
    TR(61);
}

typedef void (*SlabFn)(SlabArgs);
SlabFn hs_select_slab(int ns, bool half);
SlabFn hs_select_slab(int ns, bool half, bool pipe);

}  // namespace hs
