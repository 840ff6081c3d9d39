// Microbenchmark: the DiT's AdaLN RMSNorm (fp32 residual row [2048] -> bf16, per-row batch
// modulation) at config 2 (3000 rows), h warm in L2, back-to-back launches: the production
// kernel's access pattern (one warp per row, 16 float4 per lane) vs a TMA-bulk variant (the
// block's rows staged in shared memory by cp.async.bulk, then normalised from smem).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr int D = 2048, ROWS = 3000, TOK = 750;

template <int MINB>
__global__ void __launch_bounds__(256, MINB) norm_warp(const float *__restrict__ h, const float *__restrict__ shift,
                                                  const float *__restrict__ scale, __nv_bfloat16 *__restrict__ out) {
    constexpr int PER = D / 32 / 4;
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= ROWS) return;
    const float4 *x = (const float4 *)(h + (int64_t)row * D);
    float4 v[PER];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        v[i] = x[lane + 32 * i];
        ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float rstd = rsqrtf(ss / D + 1e-6f);
    const int b = row / TOK;
    const float4 *sh = (const float4 *)(shift + b * 6 * D), *sc = (const float4 *)(scale + b * 6 * D);
    uint2 *o = (uint2 *)(out + (int64_t)row * D);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const float4 s = sc[lane + 32 * i], t = sh[lane + 32 * i];
        float4 y = make_float4(v[i].x * rstd * (1.f + s.x) + t.x, v[i].y * rstd * (1.f + s.y) + t.y,
                               v[i].z * rstd * (1.f + s.z) + t.z, v[i].w * rstd * (1.f + s.w) + t.w);
        __nv_bfloat162 p0 = __floats2bfloat162_rn(y.x, y.y), p1 = __floats2bfloat162_rn(y.z, y.w);
        o[lane + 32 * i] = make_uint2(*(uint32_t *)&p0, *(uint32_t *)&p1);
    }
}

// TMA bulk: 4 rows per 128-thread block (one warp per row), rows staged in smem by one thread
__global__ void __launch_bounds__(128) norm_bulk(const float *__restrict__ h, const float *__restrict__ shift,
                                                  const float *__restrict__ scale, __nv_bfloat16 *__restrict__ out) {
    __shared__ __align__(128) float sx[4][D];
    __shared__ __align__(8) uint64_t bar;
    const int r0 = blockIdx.x * 4, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nr = ROWS - r0 < 4 ? ROWS - r0 : 4;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(nr * D * 4));
        for (int r = 0; r < nr; ++r)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"((uint32_t)__cvta_generic_to_shared(sx[r])), "l"(h + (int64_t)(r0 + r) * D), "r"(D * 4), "r"(sb)
                         : "memory");
    }
    __syncthreads();
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(sb)
                 : "memory");
    if (w >= nr) return;
    const int row = r0 + w;
    constexpr int PER = D / 32 / 4;
    const float4 *x = (const float4 *)sx[w];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const float4 v = x[lane + 32 * i];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float rstd = rsqrtf(ss / D + 1e-6f);
    const int b = row / TOK;
    const float4 *sh = (const float4 *)(shift + b * 6 * D), *sc = (const float4 *)(scale + b * 6 * D);
    uint2 *o = (uint2 *)(out + (int64_t)row * D);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const float4 v = x[lane + 32 * i], s = sc[lane + 32 * i], t = sh[lane + 32 * i];
        float4 y = make_float4(v.x * rstd * (1.f + s.x) + t.x, v.y * rstd * (1.f + s.y) + t.y,
                               v.z * rstd * (1.f + s.z) + t.z, v.w * rstd * (1.f + s.w) + t.w);
        __nv_bfloat162 p0 = __floats2bfloat162_rn(y.x, y.y), p1 = __floats2bfloat162_rn(y.z, y.w);
        o[lane + 32 * i] = make_uint2(*(uint32_t *)&p0, *(uint32_t *)&p1);
    }
}

// the production kernel's body (rf_dit.cu rf_dit_norm_mod<2048>: modulation loads after the reduction)
__global__ void __launch_bounds__(256) norm_prod(const float *__restrict__ h, const float *__restrict__ shift,
                                                 const float *__restrict__ scale, __nv_bfloat16 *__restrict__ out) {
    constexpr int PER = D / 32 / 4;
    const int64_t row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= ROWS) return;
    const float4 *x = (const float4 *)(h + row * D);
    float4 v[PER];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        v[i] = x[lane + 32 * i];
        ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float rstd = rsqrtf(ss / D + 1e-6f);
    const int64_t b = row / TOK;
    const float4 *sh = (const float4 *)(shift + b * 6 * D);
    const float4 *sc = (const float4 *)(scale + b * 6 * D);
    uint2 *o = (uint2 *)(out + row * D);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        float4 y = make_float4(v[i].x * rstd, v[i].y * rstd, v[i].z * rstd, v[i].w * rstd);
        const float4 s = sc[lane + 32 * i];
        y.x *= 1.f + s.x; y.y *= 1.f + s.y; y.z *= 1.f + s.z; y.w *= 1.f + s.w;
        const float4 t = sh[lane + 32 * i];
        y.x += t.x; y.y += t.y; y.z += t.z; y.w += t.w;
        __nv_bfloat162 p0 = __floats2bfloat162_rn(y.x, y.y), p1 = __floats2bfloat162_rn(y.z, y.w);
        o[lane + 32 * i] = make_uint2(*(uint32_t *)&p0, *(uint32_t *)&p1);
    }
}

// two passes over the row: sum of squares, then the row re-read (L1 / L2 hit) and scaled --
// fewer live registers (4 blocks of 256 per SM: 3000 rows in one wave)
__global__ void __launch_bounds__(256, 4) norm_2pass(const float *__restrict__ h, const float *__restrict__ shift,
                                                      const float *__restrict__ scale, __nv_bfloat16 *__restrict__ out) {
    constexpr int PER = D / 32 / 4;
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= ROWS) return;
    const float4 *x = (const float4 *)(h + (int64_t)row * D);
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const float4 v = x[lane + 32 * i];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float rstd = rsqrtf(ss / D + 1e-6f);
    const int b = row / TOK;
    const float4 *sh = (const float4 *)(shift + b * 6 * D), *sc = (const float4 *)(scale + b * 6 * D);
    uint2 *o = (uint2 *)(out + (int64_t)row * D);
#pragma unroll 4
    for (int i = 0; i < PER; ++i) {
        const float4 v = x[lane + 32 * i], s = sc[lane + 32 * i], t = sh[lane + 32 * i];
        float4 y = make_float4(v.x * rstd * (1.f + s.x) + t.x, v.y * rstd * (1.f + s.y) + t.y,
                               v.z * rstd * (1.f + s.z) + t.z, v.w * rstd * (1.f + s.w) + t.w);
        __nv_bfloat162 p0 = __floats2bfloat162_rn(y.x, y.y), p1 = __floats2bfloat162_rn(y.z, y.w);
        o[lane + 32 * i] = make_uint2(*(uint32_t *)&p0, *(uint32_t *)&p1);
    }
}

int main() {
    float *h, *mod;
    __nv_bfloat16 *out;
    cudaMalloc(&h, (size_t)ROWS * D * 4);
    cudaMalloc(&mod, (size_t)4 * 6 * D * 4);
    cudaMalloc(&out, (size_t)ROWS * D * 2);
    cudaMemset(h, 0, (size_t)ROWS * D * 4);
    cudaMemset(mod, 0, (size_t)4 * 6 * D * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&](int k) {
        if (k == 0) norm_warp<1><<<(ROWS + 7) / 8, 256>>>(h, mod, mod + D, out);
        else if (k == 1) norm_bulk<<<(ROWS + 3) / 4, 128>>>(h, mod, mod + D, out);
        else if (k == 2) norm_warp<3><<<(ROWS + 7) / 8, 256>>>(h, mod, mod + D, out);
        else if (k == 3) norm_2pass<<<(ROWS + 7) / 8, 256>>>(h, mod, mod + D, out);
        else norm_prod<<<(ROWS + 7) / 8, 256>>>(h, mod, mod + D, out);
    };
    const char *names[5] = {"warp/row, all loads hoisted", "TMA bulk rows", "warp/row, <=80 regs (3 blk/SM)",
                            "warp/row, two passes (4 blk/SM)", "production body (rf_dit_norm_mod)"};
    for (int rep = 0; rep < 2; ++rep)
    for (int k = 0; k < 5; ++k) {
        for (int it = 0; it < 10; ++it) launch(k);
        cudaEventRecord(a);
        for (int it = 0; it < 50; ++it) launch(k);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-34s: %.2f us per launch (%.0f GB/s of h read + out write)\n", names[k], ms * 1e3 / 50,
               (double)ROWS * D * 6 / (ms * 1e-3 / 50) / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
