// Packed FP32x2 FMA (FFMA2, sm_100a) throughput probe: distinct register
// operands vs broadcast scalar operand.  Prints TFLOP/s (2 FLOP per lane-op).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_probe tools/ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float lo, float hi)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

template <int MODE>
__global__ void __launch_bounds__(256) k(float *out, int iters, float a, float b)
{
    unsigned long long x[8], y[8], z[8];
    const float t = threadIdx.x * 1e-3f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = pk(t + i, t - i);
        y[i] = pk(a + t * i * 1e-7f, a - t * i * 1e-7f);
        z[i] = pk(b + t * i * 1e-9f, b);
    }
    const float s = a + t * 1e-9f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0)  // 3 distinct pairs
                    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(x[i]) : "l"(y[i]), "l"(z[(i + j) & 7]));
                if (MODE == 1) {  // scalar broadcast times a pair (complex-MAC shape)
                    const unsigned long long sb = pk(s, s);
                    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(x[i]) : "l"(sb), "l"(y[(i + j) & 7]));
                }
            }
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
        acc += lo + hi;
    }
    if (acc == 1.2345f) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
double run(float *out, int sms)
{
    const int blocks = sms * 8, threads = 256, iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MODE><<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k<MODE><<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return 4.0 * blocks * threads * (double)iters * 16 * 8 / (best * 1e-3) / 1e12;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
    printf("ffma2 distinct   %.1f TFLOP/s\n", run<0>(out, sms));
    printf("ffma2 broadcast  %.1f TFLOP/s\n", run<1>(out, sms));
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
