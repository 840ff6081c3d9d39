// Microbenchmark: scalar FFMA / DFMA throughput per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void chains(T *out, T a, T b, int iters) {
    T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <typename T>
void run(const char *name) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    T *out; cudaMalloc(&out, sizeof(T) * sms * 4 * 1024);
    int iters = 4096;
    chains<T><<<sms * 4, 1024>>>(out, (T)0.999, (T)0.001, 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    chains<T><<<sms * 4, 1024>>>(out, (T)0.999, (T)0.001, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * iters * (double)sms * 4 * 1024;
    printf("%s: %.2f TFLOP/s (%.1f FMA/clk/SM at 1.965 GHz)\n", name, flops / ms / 1e9,
           flops / 2 / (ms * 1e-3) / sms / 1.965e9);
}
int main() { run<float>("FFMA"); run<double>("DFMA"); return 0; }
