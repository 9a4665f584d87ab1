// FFMA issue-rate probe on the GPU (operand forms): register / constant /
// immediate operands, with and without operand reuse.  Prints TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_probe tools/ffma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(float *out, int iters, float a, float b)
{
    float x[8], y[8], z[8];
    const float t = threadIdx.x * 1e-3f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = t + i;
        y[i] = a + t * (i + 1) * 1e-7f;
        z[i] = b + t * (i + 2) * 1e-9f;
    }
    const float ra = a + t * 1e-9f, rb = b + t * 1e-12f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0) x[i] = fmaf(x[i], a, b);            // constant-bank operands
                if (MODE == 1) x[i] = fmaf(x[i], 0.999999f, 1e-7f);  // immediates
                if (MODE == 2) x[i] = fmaf(x[i], ra, rb);          // shared register operands
                if (MODE == 3) x[i] = fmaf(y[i], z[i], x[i]);      // 3 distinct registers
                if (MODE == 4) x[i] = fmaf(y[i], z[(i + j) & 7], x[i]);  // complex-MAC-like
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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
    return 2.0 * blocks * threads * (double)iters * 16 * 8 / (best * 1e-3) / 1e12;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
    printf("const-bank   %.1f TFLOP/s\n", run<0>(out, sms));
    printf("immediate    %.1f TFLOP/s\n", run<1>(out, sms));
    printf("shared regs  %.1f TFLOP/s\n", run<2>(out, sms));
    printf("3 distinct   %.1f TFLOP/s\n", run<3>(out, sms));
    printf("cmac-like    %.1f TFLOP/s\n", run<4>(out, sms));
    return 0;
}
