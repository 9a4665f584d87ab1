// umma_probe.cu -- checks the tcgen05 encodings the full-pass tensor-core
// kernel relies on (kind::tf32, SWIZZLE_NONE canonical layouts, TMEM
// alloc / ld / st, commit -> mbarrier), against a CPU product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe tools/umma_probe.cu
//
// T1  D[128x64]  = A[128xK] B[64xK]^T          A, B K-major in shared memory
// T2  D[128x112] = A[128xK] B2[Kx112]          B2 MN-major (same bytes as a
//                                               K-major [112-row] operand would
//                                               not be: 4 MN x 8 K core matrices)
// T3  D[128x64]  = A_tmem[128xK] B[64xK]^T     A from TMEM (tcgen05.st)
// T4  D         -= A B^T                       a_negate bit
//
// Last run on a B200 (round 1): T1, T3, T4 ok; T2 FAILS -- the MN-major
// operand encoding tried here is wrong, so the kernels use K-major operands
// only (hs_umma.cuh).  a_negate with A in shared memory (the forward pass)
// is covered by the GPU parity tests rather than by this probe.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int M = 128, K = 16, N1 = 64, N2 = 112;
#ifndef MNVAR
#define MNVAR 0
#endif

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;  // version (sm100)
    return d;                // base offset 0, SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, int a_mn, int b_mn, int a_neg)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_neg << 13) | ((uint32_t)a_mn << 15) |
           ((uint32_t)b_mn << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t tc, uint64_t da, uint64_t db, uint32_t id, int acc)
{
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tc),
                 "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t tc, uint32_t ta, uint64_t db, uint32_t id, int acc)
{
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tc),
                 "r"(ta), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_wait(uint64_t *bar, uint32_t &phase)
{
    if (threadIdx.x == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(bar)) : "memory");
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major canonical offset (bytes): 8-row x 16-byte core matrices,
// rows-groups at SBO = 128, k-quads at LBO = rows/8 * 128
__device__ __forceinline__ uint32_t kmaj(int row, int k, int rows)
{
    return (row >> 3) * 128 + (k >> 2) * (rows / 8) * 128 + (row & 7) * 16 + (k & 3) * 4;
}
// MN-major canonical offset: 4 MN x 8 K core matrices, MN-quads at SBO = 128 *
// (K/8), K-octets at LBO = 128
__device__ __forceinline__ uint32_t mnmaj(int n, int k)
{
    return (n >> 2) * 128 * (K / 8) + (k >> 3) * 128 + (k & 7) * 16 + (n & 3) * 4;
}

__global__ void probe(const float *A, const float *B, const float *B2, float *D1, float *D2, float *D3, float *D4)
{
    __shared__ __align__(1024) float sA[M * K];
    __shared__ __align__(1024) float sB[N1 * K];
    __shared__ __align__(1024) float sB2[N2 * K];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    char *pa = reinterpret_cast<char *>(sA), *pb = reinterpret_cast<char *>(sB), *pb2 = reinterpret_cast<char *>(sB2);
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<float *>(pa + kmaj(r, k, M)) = A[i];
    }
    for (int i = tid; i < N1 * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<float *>(pb + kmaj(r, k, N1)) = B[i];
    }
    for (int i = tid; i < K * N2; i += blockDim.x) {  // B2[k][n]
        const int k = i / N2, n = i % N2;
        *reinterpret_cast<float *>(pb2 + mnmaj(n, k)) = B2[i];
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
    uint32_t phase = 0;
    const uint32_t aA = smem_u32(sA), aB = smem_u32(sB), aB2 = smem_u32(sB2);
    // T1 at columns [0,64), T2 at [64,176), T3 at [176,240), T4 at [240,304)
    // TMEM A operand for T3 at [320, 336)
    {   // stage A into TMEM: thread = row (lane), 16 columns
        float v[K];
        for (int k = 0; k < K; ++k) v[k] = A[tid * K + k];
        const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + 320;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(ta), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
                     "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        for (int ks = 0; ks < K / 8; ++ks) {
            const uint64_t da = sdesc(aA + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
            const uint64_t db = sdesc(aB + ks * 2 * (N1 / 8) * 128, (N1 / 8) * 128, 128);
            const int v = MNVAR;
            const uint64_t db2 = (v & 1) ? sdesc(aB2 + ks * 128, 128 * (K / 8), 128) : sdesc(aB2 + ks * 128, 128, 128 * (K / 8));
            mma_ss(tm + 0, da, db, idesc_tf32(M, N1, 0, 0, 0), ks);
            mma_ss(tm + 64, da, db2, idesc_tf32(M, (v & 2) ? 64 : N2, 0, 1, 0), ks);
            mma_ts(tm + 176, tm + 320 + ks * 8, db, idesc_tf32(M, N1, 0, 0, 0), ks);
            mma_ss(tm + 240, da, db, idesc_tf32(M, N1, 0, 0, 0), ks);
        }
        for (int ks = 0; ks < K / 8; ++ks) {  // T4: D -= A B^T -> 0
            const uint64_t da = sdesc(aA + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
            const uint64_t db = sdesc(aB + ks * 2 * (N1 / 8) * 128, (N1 / 8) * 128, 128);
            mma_ts(tm + 240, tm + 320 + ks * 8, db, idesc_tf32(M, N1, 0, 0, 1), 1);
        }
    }
    __syncwarp();
    commit_wait(&bar, phase);
    const uint32_t lane_base = tm + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 304; c += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(lane_base + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 16; ++j) {
            const int col = c + j;
            const float f = __uint_as_float(v[j]);
            if (col < 64) D1[tid * N1 + col] = f;
            else if (col < 176) D2[tid * N2 + col - 64] = f;
            else if (col < 240) D3[tid * N1 + col - 176] = f;
            else D4[tid * N1 + col - 240] = f;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main()
{
    std::vector<float> A(M * K), B(N1 * K), B2(K * N2);
    srand(1);
    auto rv = []() { return (float)((rand() % 17) - 8) * 0.25f; };
    for (auto &x : A) x = rv();
    for (auto &x : B) x = rv();
    for (auto &x : B2) x = rv();
    float *dA, *dB, *dB2, *d1, *d2, *d3, *d4;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dB2, B2.size() * 4));
    CK(cudaMalloc(&d1, M * N1 * 4)); CK(cudaMalloc(&d2, M * N2 * 4)); CK(cudaMalloc(&d3, M * N1 * 4)); CK(cudaMalloc(&d4, M * N1 * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB2, B2.data(), B2.size() * 4, cudaMemcpyHostToDevice));
    probe<<<1, 128>>>(dA, dB, dB2, d1, d2, d3, d4);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> h1(M * N1), h2(M * N2), h3(M * N1), h4(M * N1);
    CK(cudaMemcpy(h1.data(), d1, h1.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), d2, h2.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h3.data(), d3, h3.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h4.data(), d4, h4.size() * 4, cudaMemcpyDeviceToHost));
    int bad1 = 0, bad2 = 0, bad3 = 0, bad4 = 0;
    for (int m = 0; m < M; ++m) {
        for (int n = 0; n < N1; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
            if (fabs(h1[m * N1 + n] - s) > 1e-6) { if (bad1 < 4) printf("T1 m=%d n=%d got %g want %g\n", m, n, h1[m * N1 + n], s); ++bad1; }
            if (fabs(h3[m * N1 + n] - s) > 1e-6) { if (bad3 < 4) printf("T3 m=%d n=%d got %g want %g\n", m, n, h3[m * N1 + n], s); ++bad3; }
            if (fabs(h4[m * N1 + n]) > 1e-6) { if (bad4 < 4) printf("T4 m=%d n=%d got %g want 0\n", m, n, h4[m * N1 + n]); ++bad4; }
        }
        for (int n = 0; n < N2; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B2[k * N2 + n];
            if ((!(MNVAR & 2) || n < 64) && fabs(h2[m * N2 + n] - s) > 1e-6) { if (bad2 < 4) printf("T2 m=%d n=%d got %g want %g\n", m, n, h2[m * N2 + n], s); ++bad2; }
        }
    }
    printf("T1 ss kmajor %s (%d bad)\nT2 ss mnmajor B %s (%d bad)\nT3 ts A in tmem %s (%d bad)\nT4 a_negate (A in tmem) %s (%d bad)\n",
           bad1 ? "FAIL" : "ok", bad1, bad2 ? "FAIL" : "ok", bad2, bad3 ? "FAIL" : "ok", bad3, bad4 ? "FAIL" : "ok", bad4);
    return (bad1 || bad2 || bad3 || bad4) ? 1 : 0;
}
