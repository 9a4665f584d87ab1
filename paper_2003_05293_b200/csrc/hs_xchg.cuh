// hs_xchg.cuh -- peer-memory exchange of group partials for the row-sharded
// solve (SURVEY.md 8(e), config 4 across GPUs), replacing the host
// round trip of hs_shard_pass / hs_shard_update.
//
// Every rank owns one exchange buffer (CUDA IPC-shared with the others):
//   flags[world]                      epoch last published by each rank
//   xbuf[2][B][ngmax][np] double2     the group partials of ALL ranks, two
//                                     pass slots (pass parity)
// Pass j on rank r:
//   1. the pass kernel over r's fold-group-aligned chunk range (ACT_NONE);
//   2. hs_publish_kernel: one CTA per (own group, pattern) folds the group's
//      chunk partials in chunk order (fp64, = hs_group_fold_kernel) and
//      stores the result into EVERY rank's xbuf over NVLink peer memory;
//      the last CTA fences (system scope) and release-stores the epoch into
//      every rank's flags[r];
//   3. hs_gather_update_kernel: acquire-spins until every flags[q] reached
//      the epoch, folds all groups in group order from the LOCAL xbuf and
//      applies the update (hs_update) -- identical on every rank and
//      bitwise equal to the single-GPU solve.
// Two slots suffice: a rank can publish pass j+2 only after its update of
// pass j+1, which needs every rank's pass j+1 publish, which each rank
// issues after its own update of pass j.  The spin is bounded (2 s of
// globaltimer), and a timeout marks the pattern failed instead of hanging
// the device.  Failure propagates: a rank with a failed pattern (timeout,
// degenerate fields) publishes its epoch with kXchgAbort set, and every peer
// whose gather sees that bit marks its patterns failed too -- all ranks stop
// together and raise together (distributed.solve_sharded all-gathers the
// status before the phase exchange) instead of folding stale partials.
#pragma once

#include "hs_kernels.cuh"

namespace hs {

struct XchgArgs {
    FoldArgs f;                 // local chunk partials, np, strides, update args
    int32_t g_lo, g_hi;         // this rank's groups
    int32_t ngroups;            // all groups of the pass
    int32_t ngmax;              // group capacity of a slot
    int32_t world, rank, slot;
    const unsigned long long *epoch0;  // device: epoch base of the current solve (hs_epoch_advance_kernel)
    int32_t pass;                      // the pass publishes / waits for epoch *epoch0 + pass + 1
    double2 *const *peer_xbuf;  // [world] xbuf bases (slot 0), device pointers
    unsigned long long *const *peer_flags;  // [world] flags bases
    unsigned long long *flags_local;
    const double2 *xbuf_local;
    int32_t *pub_cnt;           // local arrival counter (self-resetting)
    int32_t announce_only;      // rank without groups: publish the epoch only
    int32_t batch;              // patterns (status entries) of this rank
};

constexpr unsigned long long kXchgAbort = 1ull << 63;   // epoch flag bit: the publisher failed
constexpr unsigned long long kXchgTimeoutNs = 2000000000ull;

__device__ __forceinline__ unsigned long long hs_globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void hs_st_release_sys(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long hs_ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Start of a sharded solve: the passes of this solve publish epochs
// base + 1 .. base + passes.  The epoch lives in device memory (not in the
// kernel arguments) so a captured solve graph replays with fresh epochs.
static __global__ void hs_epoch_advance_kernel(unsigned long long *ctr, unsigned long long *base, int passes)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *base = *ctr;
        *ctr += (unsigned long long)passes;
    }
}

static __global__ void __launch_bounds__(128) hs_publish_kernel(const XchgArgs a)
{
    const int grp = a.g_lo + blockIdx.x, pat = blockIdx.y, np = a.f.np;
    const int c0 = grp * kGroup, c1 = min(c0 + kGroup, a.f.nchunks);
    const float2 *part = a.f.partials + (int64_t)pat * a.f.part_stride;
    const int64_t off = (((int64_t)a.slot * gridDim.y + pat) * a.ngmax + grp) * np;
    for (int k = threadIdx.x; k < (a.announce_only ? 0 : np); k += blockDim.x) {
        double sx = 0.0, sy = 0.0;
        for (int c = c0; c < c1; ++c) {
            const float2 v = __ldcg(part + (int64_t)c * np + k);
            sx += (double)v.x;
            sy += (double)v.y;
        }
        const double2 g = make_double2(sx, sy);
        for (int r = 0; r < a.world; ++r) a.peer_xbuf[r][off + k] = g;  // NVLink peer stores
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int total = (int)(gridDim.x * gridDim.y);
        if (atomicAdd(a.pub_cnt, 1) == total - 1) {
            *a.pub_cnt = 0;
            __threadfence_system();
            bool failed = false;   // any pattern of this rank failed: tell the peers
            for (int b = 0; b < a.batch; ++b) failed |= (*(volatile int32_t *)(a.f.u.status + b) != 0);
            const unsigned long long epoch = *a.epoch0 + (unsigned long long)a.pass + 1ull;
            const unsigned long long v = epoch | (failed ? kXchgAbort : 0ull);
            for (int r = 0; r < a.world; ++r) hs_st_release_sys(a.peer_flags[r] + a.rank, v);
        }
    }
}

static __global__ void __launch_bounds__(kThreads) hs_gather_update_kernel(const XchgArgs a)
{
    __shared__ double dbuf[kThreads];
    __shared__ int ibuf[kThreads];
    __shared__ int s_ok;
    extern __shared__ double2 Eu[];  // [np] fields + [2 np] scratch
    const int pat = blockIdx.x, np = a.f.np;
    if (threadIdx.x == 0) {
        int ok = 1;
        const unsigned long long epoch = *a.epoch0 + (unsigned long long)a.pass + 1ull;
        const unsigned long long t0 = hs_globaltimer();
        for (int r = 0; r < a.world && ok; ++r) {
            unsigned long long v;
            while (((v = hs_ld_acquire_sys(a.flags_local + r)) & ~kXchgAbort) < epoch) {
                __nanosleep(128);
                if (hs_globaltimer() - t0 > kXchgTimeoutNs) {  // a peer never published
                    ok = 0;
                    break;
                }
            }
            if (v & kXchgAbort) ok = 0;  // a peer failed this pass
        }
        s_ok = ok;
    }
    __syncthreads();
    if (!s_ok) {
        if (threadIdx.x == 0) a.f.u.status[pat] = 5;  // HS_ECUDA: exchange timed out or a peer failed
        return;
    }
    if (a.f.u.status[pat] != 0) return;
    const double2 *gp = a.xbuf_local + (((int64_t)a.slot * gridDim.x + pat) * a.ngmax) * np;
    for (int k = threadIdx.x; k < np; k += kThreads) {
        double sx = 0.0, sy = 0.0;
        for (int g = 0; g < a.ngroups; ++g) {
            const double2 v = __ldcv(gp + (int64_t)g * np + k);
            sx += v.x;
            sy += v.y;
        }
        Eu[k] = make_double2(sx, sy);
    }
    __syncthreads();
    hs_update(a.f.u, pat, Eu, reinterpret_cast<double *>(Eu + np), dbuf, ibuf);
}

}  // namespace hs
