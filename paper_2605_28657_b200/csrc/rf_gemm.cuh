// Persistent warp-specialised tcgen05 GEMM for sm_100a:  D[M,N] = A[M,K] * B[N,K]^T
// (bf16 operands, both K-major as nn.Linear stores them; fp32 accumulation in TMEM).
//
//   warp 0   : TMA producer (one elected lane) -- A/B tiles into a STAGES-deep ring of
//              SWIZZLE_128B shared-memory buffers, completion via mbarrier tx counts
//   warp 1   : MMA issuer (one elected lane) -- BK/16 tcgen05.mma (M=128, N=BN, K=16)
//              per stage into one of two TMEM accumulators; tcgen05.commit frees the
//              smem stage and, after the last k block, hands the accumulator over
//   warps 2-5: epilogue -- tcgen05.ld 32 columns at a time, fused epilogue, global store,
//              then release the accumulator so the MMA warp can start tile i+2
// The two accumulators (2 x BN TMEM columns) let the epilogue of tile i overlap the
// main loop of tile i+1.  Tiles are walked m-fastest so CTAs running concurrently share
// the same B (weight) tile through L2.
#pragma once
#include "rf_sm100.cuh"

namespace rf::gemm {

enum Epi : int {
    kStoreBF16 = 0,   // out(bf16)[m,n] = acc
    kStoreF32 = 1,    // out(f32)[m,n] = acc
    kResidGate = 2,   // out(f32)[m,n] += gate[m / rows_per_batch, n] * acc   (AdaLN gated residual)
    kSwiGLU = 3,      // columns interleaved (g, u): out(bf16)[m, n/2] = silu(g) * u
    kStoreF32Scale = 4,  // out(f32)[m,n] = alpha * acc
    kBF16Rope = 5,    // out(bf16)[m,n] = acc, interleaved-pair RoPE on columns < rope_cols
};

struct EpiArgs {
    void *out;
    int64_t ldo;            // elements
    const float *gate;      // kResidGate
    int64_t gate_ld;        // elements between batches of gate
    int rows_per_batch;
    float alpha;
    const float2 *rope;     // kBF16Rope: (cos, sin)[pos * 64 + pair], pos = m % rows_per_batch
    int rope_cols;
    // kBF16Rope: columns >= vt_col0 (the V heads) are written transposed instead, to
    // vt[((b * vt_heads + hv) * 128 + dim) * vt_ld + pos] (b = m / rows_per_batch) -- the
    // K-major B operand of the attention's P V^T product.
    __nv_bfloat16 *vt;
    int vt_col0, vt_heads;
    int64_t vt_ld;
};

constexpr int BM = 128, BK = 64;
template <int BN>
struct Cfg {
    static constexpr int STAGES = BN == 256 ? 4 : 6;
    static constexpr uint32_t A_BYTES = BM * BK * 2;
    static constexpr uint32_t B_BYTES = BN * BK * 2;
    static constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + 256;
};

__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16(x)); }

template <int BN, int EPI>
__global__ void __launch_bounds__(192, 1)
rf_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, int M,
               int N, int K, EpiArgs epi) {
    using namespace rf::sm100;
    using C = Cfg<BN>;
    constexpr int STAGES = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = base;
    uint8_t *sB = base + STAGES * C::A_BYTES;
    uint64_t *full = (uint64_t *)(sB + STAGES * C::B_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc<2 * BN>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int num_m = (M + BM - 1) / BM, num_n = N / BN, kblocks = K / BK;
    const int num_tiles = num_m * num_n;

    if (warp == 0) {
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                const int m0 = (t % num_m) * BM, n0 = (t / num_m) * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
                    tma_load_2d(sA + stage * C::A_BYTES, &tma_a, &full[stage], kb * BK, m0);
                    tma_load_2d(sB + stage * C::B_BYTES, &tma_b, &full[stage], kb * BK, n0);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + acc * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = sdesc_sw128(sA + stage * C::A_BYTES);
                    const uint64_t bd = sdesc_sw128(sB + stage * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc,
                                  (kb | k) != 0);
                    umma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const int m0 = (t % num_m) * BM, n0 = (t / num_m) * BN;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int m = m0 + q * 32 + lane;
            const bool live = m < M;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), r);
                tmem_ld_wait();
                if (!live) continue;
                const int n = n0 + c0;
                if constexpr (EPI == kStoreBF16) {
                    __nv_bfloat16 *o = (__nv_bfloat16 *)epi.out + (int64_t)m * epi.ldo + n;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        uint4 pk;
                        uint32_t *p = (uint32_t *)&pk;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[v * 8 + 2 * e]),
                                                                     __uint_as_float(r[v * 8 + 2 * e + 1]));
                            p[e] = *(uint32_t *)&h;
                        }
                        *(uint4 *)(o + v * 8) = pk;
                    }
                } else if constexpr (EPI == kBF16Rope) {
                    if (epi.vt && n >= epi.vt_col0) {
                        const int cv = n - epi.vt_col0, hv = cv >> 7, dim0 = cv & 127;
                        const int64_t b = m / epi.rows_per_batch, pos = m % epi.rows_per_batch;
                        __nv_bfloat16 *dst = epi.vt + ((b * epi.vt_heads + hv) * 128 + dim0) * epi.vt_ld + pos;
#pragma unroll
                        for (int e = 0; e < 32; ++e)   // lanes hold consecutive tokens: coalesced
                            dst[(int64_t)e * epi.vt_ld] = __float2bfloat16(__uint_as_float(r[e]));
                        continue;
                    }
                    __nv_bfloat16 *o = (__nv_bfloat16 *)epi.out + (int64_t)m * epi.ldo + n;
                    const bool rot = n < epi.rope_cols;
                    const float2 *cs = epi.rope + (int64_t)(m % epi.rows_per_batch) * 64 + ((n & 127) >> 1);
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        uint4 pk;
                        uint32_t *p = (uint32_t *)&pk;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float x0 = __uint_as_float(r[v * 8 + 2 * e]), x1 = __uint_as_float(r[v * 8 + 2 * e + 1]);
                            if (rot) {
                                // q/k are bf16 Linear outputs: round, then rotate in fp32
                                x0 = bf16_round(x0);
                                x1 = bf16_round(x1);
                                const float2 c = cs[v * 4 + e];
                                const float y0 = x0 * c.x - x1 * c.y, y1 = x0 * c.y + x1 * c.x;
                                x0 = y0;
                                x1 = y1;
                            }
                            __nv_bfloat162 hh = __floats2bfloat162_rn(x0, x1);
                            p[e] = *(uint32_t *)&hh;
                        }
                        *(uint4 *)(o + v * 8) = pk;
                    }
                } else if constexpr (EPI == kStoreF32 || EPI == kStoreF32Scale) {
                    float *o = (float *)epi.out + (int64_t)m * epi.ldo + n;
                    const float a = EPI == kStoreF32Scale ? epi.alpha : 1.0f;
#pragma unroll
                    for (int v = 0; v < 8; ++v)
                        *(float4 *)(o + v * 4) = make_float4(a * __uint_as_float(r[4 * v]), a * __uint_as_float(r[4 * v + 1]),
                                                             a * __uint_as_float(r[4 * v + 2]),
                                                             a * __uint_as_float(r[4 * v + 3]));
                } else if constexpr (EPI == kResidGate) {
                    float *o = (float *)epi.out + (int64_t)m * epi.ldo + n;
                    const float *g = epi.gate + (int64_t)(m / epi.rows_per_batch) * epi.gate_ld + n;
                    // all loads first (out and gate may alias as far as the compiler knows,
                    // which would otherwise serialise one DRAM round trip per float4)
                    float4 xv[8], gv[8];
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        xv[v] = __ldcs((const float4 *)(o + v * 4));
                        gv[v] = __ldg((const float4 *)(g + v * 4));
                    }
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        float4 x = xv[v];
                        x.x += gv[v].x * __uint_as_float(r[4 * v]);
                        x.y += gv[v].y * __uint_as_float(r[4 * v + 1]);
                        x.z += gv[v].z * __uint_as_float(r[4 * v + 2]);
                        x.w += gv[v].w * __uint_as_float(r[4 * v + 3]);
                        *(float4 *)(o + v * 4) = x;
                    }
                } else if constexpr (EPI == kSwiGLU) {
                    __nv_bfloat16 *o = (__nv_bfloat16 *)epi.out + (int64_t)m * epi.ldo + n / 2;
                    uint4 pk[2];
                    uint32_t *p = (uint32_t *)pk;
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        float y[2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            // gate/up rounded to bf16 like a bf16 Linear output, then SiLU(g)*u
                            const float gt = bf16_round(__uint_as_float(r[4 * e + 2 * h]));
                            const float up = bf16_round(__uint_as_float(r[4 * e + 2 * h + 1]));
                            y[h] = gt / (1.0f + __expf(-gt)) * up;
                        }
                        __nv_bfloat162 hh = __floats2bfloat162_rn(y[0], y[1]);
                        p[e] = *(uint32_t *)&hh;
                    }
                    *(uint4 *)o = pk[0];
                    *(uint4 *)(o + 8) = pk[1];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    __syncthreads();
    if (warp == 1) tmem_dealloc<2 * BN>(tmem);
}

}  // namespace rf::gemm
