// FP64 DFMA throughput probe (B200 keeps a real FP64 pipe; the B300 notes'
// "vestigial FP64" is sm_103a only).  Prints TFLOP/s for dependent-chain
// DFMA streams with register / shared operands, next to the FFMA figure.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_probe tools/dfma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int MODE>
__global__ void __launch_bounds__(256) k(T *out, int iters, T a, T b)
{
    T x[8], y[8], z[8];
    const T t = threadIdx.x * (T)1e-3;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = t + i;
        y[i] = a + t * (i + 1) * (T)1e-7;
        z[i] = b + t * (i + 2) * (T)1e-9;
    }
    const T ra = a + t * (T)1e-9, rb = b + t * (T)1e-12;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0) x[i] = fma(x[i], ra, rb);
                if (MODE == 1) x[i] = fma(y[i], z[(i + j) & 7], x[i]);
            }
        }
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == (T)1.2345) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename T, int MODE>
double run(T *out, int sms, int per_sm)
{
    const int blocks = sms * per_sm, threads = 256, iters = 1024;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<T, MODE><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k<T, MODE><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
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
    double *out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
    for (int per_sm : {2, 4, 8}) {
        printf("blocks/SM %d: DFMA shared-operand %.2f TFLOP/s, DFMA cmac-like %.2f TFLOP/s, "
               "FFMA shared-operand %.2f TFLOP/s\n", per_sm,
               run<double, 0>(out, sms, per_sm), run<double, 1>(out, sms, per_sm),
               run<float, 0>((float *)out, sms, per_sm));
    }
    return 0;
}
