// Microbenchmark: MUFU.EX2 (ex2.approx.ftz.f32) throughput per SM, at full occupancy and
// with only 1-2 warps per SM sub-partition (the attention softmax's configuration).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <int ILP>
__global__ void chains(float *out, float a, int iters) {
    float x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = -1.f - 0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = ex2(x[i]) * a - 1.f;   // MUFU + FFMA per element
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP>
void run(int blocks_per_sm, int threads) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; cudaMalloc(&out, sizeof(float) * sms * blocks_per_sm * threads);
    int iters = 2048;
    chains<ILP><<<sms * blocks_per_sm, threads>>>(out, 0.5f, 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    chains<ILP><<<sms * blocks_per_sm, threads>>>(out, 0.5f, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = (double)ILP * iters * sms * blocks_per_sm * threads;
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("ILP %2d, %4d threads/SM: %.2f ex2/clk/SM (at %.0f MHz nominal), %.1f cycles per warp-instr per SMSP\n", ILP,
           blocks_per_sm * threads, ops / cyc / sms, clk / 1e3,
           cyc / ((double)ILP * iters * blocks_per_sm * threads / 32 / 4));
    cudaFree(out);
}
int main() {
    run<8>(4, 512);
    run<16>(1, 128);
    run<16>(1, 256);
    run<32>(1, 256);
    run<16>(1, 512);
    return 0;
}
