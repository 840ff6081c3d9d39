// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M = 128) throughput per SM for
// N = 64 / 128 / 256, A from shared memory (SS) or from TMEM (TS).  One CTA per SM, one
// thread issues back-to-back MMAs (K = 16 each) into TMEM, commits once and waits.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "rf_sm100.cuh"
using namespace rf::sm100;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) umma_loop(int iters, unsigned long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t *base = (uint8_t *)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t *)base)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_bf16(128, N);
        const uint64_t ad = sdesc_sw128(base), bd = sdesc_sw128(base + 32768);
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if constexpr (TS)
                    umma_bf16_ts(tmem + 256, tmem + (k & 7) * 8, bd + (uint64_t)((k & 3) * 2), idesc, 1u);
                else
                    umma_bf16(tmem + 256, ad + (uint64_t)((k & 3) * 2), bd + (uint64_t)((k & 3) * 2), idesc, 1u);
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0) *cyc = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
void run(const char *name) {
    unsigned long long *d, h;
    cudaMalloc(&d, 8);
    auto k = umma_loop<N, TS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k<<<sms, 128, 66 * 1024>>>(16, d);
    cudaDeviceSynchronize();
    const int iters = 2048;
    k<<<sms, 128, 66 * 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double mmas = 16.0 * iters, flop = 2.0 * 128 * N * 16;
    printf("%-16s %s: %.1f cycles per MMA, %.0f FLOP/cycle/SM\n", name, cudaGetErrorString(e), (double)h / mmas,
           flop * mmas / (double)h);
    cudaFree(d);
}

int main() {
    run<64, false>("M128 N64  SS");
    run<128, false>("M128 N128 SS");
    run<256, false>("M128 N256 SS");
    run<64, true>("M128 N64  TS");
    run<128, true>("M128 N128 TS");
    run<256, true>("M128 N256 TS");
    return 0;
}
