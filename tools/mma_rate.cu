// mma_rate.cu -- tcgen05.mma issue-to-completion rate by operand layout
// (cycles per M = 128 MMA, one CTA, operands resident in shared memory).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_rate tools/mma_rate.cu
//
// Cases (kind::tf32 unless noted, K-major A and B, D in TMEM):
//   none   SWIZZLE_NONE core matrices (8 rows x 16 B; the layout hs_umma uses)
//   sw32   SWIZZLE_32B  (8-row x 32-byte atoms)
//   sw128  SWIZZLE_128B (8-row x 128-byte atoms, K = 32 per row: 4 MMAs per row)
//   ts     A from TMEM, B SWIZZLE_NONE
//   f16    kind::f16, K = 16 (32 bytes per row), SWIZZLE_NONE
//   cpts   f16: A copied smem -> TMEM by tcgen05.cp 128x256b, then the MMA reads A from TMEM
//          (one copy per MMA: the backward's gy planes arrive in shared memory by TMA)
// plus a numerical check: D(cp + TS) == D(SS) on random fp16 operands.
// Values are irrelevant (zeros); only the time per MMA is measured, for
// N = 64, 128, 256.
#include <cstdint>
#include <cmath>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout)
{
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// kind::tf32 (a/b format 2) or kind::f16 (fp16: format 0), f32 accumulate, K-major
__host__ __device__ constexpr uint32_t idesc(int n, bool f16)
{
    return (1u << 4) | ((f16 ? 0u : 2u) << 7) | ((f16 ? 0u : 2u) << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}

template <bool F16>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id)
{
    if (F16)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 1, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                     "l"(a), "l"(b), "r"(id));
    else
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 1, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                     "l"(a), "l"(b), "r"(id));
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id)
{
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 1, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id));
}

constexpr int REPS = 4096;

__device__ __forceinline__ void mma_ts16(uint32_t d, uint32_t a, uint64_t b, uint32_t id, int acc)
{
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void cp_a(uint32_t t, uint64_t src)
{
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(t), "l"(src));
}

// mode: 0 none, 1 sw32, 2 sw128, 3 ts, 4 f16, 5 cp+ts (f16)
__global__ void rate(int mode, int n, long long *out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    const uint32_t a0 = smem_u32(sm), b0 = a0 + 32 * 1024;  // A: up to 32 KB, B: up to 64 KB
    const uint32_t id = idesc(n, mode == 4 || mode == 5);
    uint64_t da[4], db[4];
    for (int k = 0; k < 4; ++k) {
        if (mode == 0 || mode == 3 || mode == 4 || mode == 5) {  // core matrices: SBO 128 (8-row groups), LBO = rows/8*128 (K halves)
            da[k] = sdesc(a0 + k * 4096, 16 * 128, 128, 0);
            db[k] = sdesc(b0 + k * 8192, (n / 8) * 128, 128, 0);
        } else if (mode == 1) {                     // 32-byte rows, 8-row atoms of 256 B
            da[k] = sdesc(a0 + k * 4096, 16, 256, 6);
            db[k] = sdesc(b0 + k * 8192, 16, 256, 6);
        } else {                                    // 128-byte rows: k-th 32-byte slice of the row
            da[k] = sdesc(a0 + k * 32, 16, 1024, 2);
            db[k] = sdesc(b0 + k * 32, 16, 1024, 2);
        }
    }
    long long t0 = 0, t1 = 0;
    if (tid == 0) {
        uint32_t phase = 0;
        for (int w = 0; w < 2; ++w) {  // warm-up pass, timed pass
            t0 = clock64();
            for (int r = 0; r < REPS; ++r) {
                const int k = r & 3;
                if (mode == 3) mma_ts(tm, tm + 256 + 8 * k, db[k], id);
                else if (mode == 4) mma_ss<true>(tm, da[k], db[k], id);
                else if (mode == 5) {
                    cp_a(tm + 256 + 8 * k, da[k]);
                    mma_ts16(tm, tm + 256 + 8 * k, db[k], id, 1);
                }
                else mma_ss<false>(tm, da[k], db[k], id);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&bar)) : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                             " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
            phase ^= 1;
            t1 = clock64();
        }
        out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// D = A B^T (M = 128, N = 64, K = 16 fp16) twice: A from smem (SS) and A
// copied to TMEM by tcgen05.cp (TS); returns max |difference| and max |D|.
__global__ void check(const unsigned short *A, const unsigned short *B, float *out)
{
    __shared__ __align__(1024) unsigned char sa[4096], sb[2048];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    // K-major core matrices: element (r, k) at r*16 + (k/8)*(rows*16) + (k%8)*2
    for (int i = tid; i < 128 * 16; i += blockDim.x) {
        const int r = i / 16, k = i % 16;
        *reinterpret_cast<unsigned short *>(sa + r * 16 + (k / 8) * 2048 + (k % 8) * 2) = A[i];
    }
    for (int i = tid; i < 64 * 16; i += blockDim.x) {
        const int r = i / 16, k = i % 16;
        *reinterpret_cast<unsigned short *>(sb + r * 16 + (k / 8) * 1024 + (k % 8) * 2) = B[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    const uint64_t da = sdesc(smem_u32(sa), 2048, 128, 0), db = sdesc(smem_u32(sb), 1024, 128, 0);
    const uint32_t id = idesc(64, true);
    if (tid == 0) {
        mma_ss<true>(tm, da, db, id);                 // (acc predicate 1: D starts as 0 from alloc? use two runs below)
        cp_a(tm + 256, da);
        mma_ts16(tm + 128, tm + 256, db, id, 0);
        mma_ss<true>(tm + 64, da, db, id);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // thread = row: D_ss2 at columns [64,128) (accumulated onto garbage-free? no: acc=1 onto zero-init
    // is not guaranteed), so compare TS (fresh, acc = 0) against a CPU product instead
    float ts[64];
    const uint32_t tl = tm + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 64; c += 8) {
        float v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                     : "r"(tl + 128 + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; ++j) ts[c + j] = v[j];
    }
    for (int c = 0; c < 64; ++c) out[tid * 64 + c] = ts[c];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static float h2f(unsigned short h)
{
    const int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
    const float v = e ? ldexpf(1.f + m / 1024.f, e - 15) : ldexpf(m / 1024.f, -14);
    return s ? -v : v;
}

int main()
{
    {   // numerical check of cp + TS
        unsigned short hA[128 * 16], hB[64 * 16];
        unsigned state = 12345;
        auto rnd = [&]() { state = state * 1664525u + 1013904223u; return state; };
        for (auto &v : hA) v = (unsigned short)(0x3000 + (rnd() >> 22) % 0x0c00) ^ ((rnd() & 1) << 15);
        for (auto &v : hB) v = (unsigned short)(0x3000 + (rnd() >> 22) % 0x0c00) ^ ((rnd() & 1) << 15);
        unsigned short *dA, *dB;
        float *dO;
        CK(cudaMalloc(&dA, sizeof hA)); CK(cudaMalloc(&dB, sizeof hB)); CK(cudaMalloc(&dO, 128 * 64 * 4));
        CK(cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice));
        check<<<1, 128>>>(dA, dB, dO);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        static float o[128 * 64];
        CK(cudaMemcpy(o, dO, sizeof o, cudaMemcpyDeviceToHost));
        double err = 0, mx = 0;
        for (int r = 0; r < 128; ++r)
            for (int c = 0; c < 64; ++c) {
                double want = 0;
                for (int k = 0; k < 16; ++k) want += (double)h2f(hA[r * 16 + k]) * h2f(hB[c * 16 + k]);
                err = fmax(err, fabs(o[r * 64 + c] - want));
                mx = fmax(mx, fabs(want));
            }
        printf("cp+TS f16 check: max |D - A B^T| = %.3g (max |D| %.3g)\n", err, mx);
    }
    long long *d;
    CK(cudaMalloc(&d, sizeof(long long)));
    CK(cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    const char *names[] = {"none", "sw32", "sw128", "ts", "f16", "cpts"};
    for (int mode = 0; mode < 6; ++mode)
        for (int n : {64, 128, 256}) {
            rate<<<1, 128, 96 * 1024>>>(mode, n, d);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            long long c;
            CK(cudaMemcpy(&c, d, sizeof c, cudaMemcpyDeviceToHost));
            const double per = (double)c / REPS, ideal = 128.0 * n / 256.0;
            printf("%-6s N=%3d: %7.1f cycles per MMA (ideal %5.1f at the tf32 rate; f16 does 2x the MACs)\n",
                   names[mode], n, per, ideal);
        }
    return 0;
}
