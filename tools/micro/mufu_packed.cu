// Microbenchmark: packed MUFU exponentials -- ex2.approx.ftz.bf16x2 and ex2.approx.f16x2 (two
// results per lane per instruction) vs ex2.approx.ftz.f32 -- results per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int KIND>
__device__ __forceinline__ uint32_t op(uint32_t x) {
    uint32_t y;
    if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=r"(y) : "r"(x));
    if (KIND == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
    if (KIND == 2) asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
template <int KIND, int ILP>
__global__ void chains(uint32_t *out, int iters) {
    uint32_t x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = KIND == 0 ? 0xbf800000u - threadIdx.x - i : 0xbf80bf80u - threadIdx.x - i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = op<KIND>(x[i]) ^ 0x80008000u;   // keep inputs negative-ish
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int KIND>
void run(const char *name, int results_per_op) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *out; cudaMalloc(&out, sizeof(uint32_t) * sms * 4 * 512);
    const int iters = 4096;
    chains<KIND, 8><<<sms * 4, 512>>>(out, 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    chains<KIND, 8><<<sms * 4, 512>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = 8.0 * iters * sms * 4 * 512;
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-22s %.2f instr/clk/SM  %.2f results/clk/SM (nominal clock)\n", name, ops / cyc / sms,
           results_per_op * ops / cyc / sms);
    cudaFree(out);
}
int main() {
    run<0>("ex2.approx.ftz.f32", 1);
    run<1>("ex2.approx.ftz.bf16x2", 2);
    run<2>("ex2.approx.f16x2", 2);
    return 0;
}
