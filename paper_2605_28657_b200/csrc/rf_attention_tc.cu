// Attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), head dim 128.
//
// Single-pass (online-softmax) flash attention, warp-specialised: a TMA warp streams K and
// V^T tiles (V written transposed by the QKV GEMM epilogue, so it is the K-major B operand
// of P V), one elected thread issues tcgen05.mma (S = Q K^T into TMEM, O += P V as a TS
// MMA with P read from TMEM), and one warpgroup per query head runs the softmax with one
// query row per thread (its S and O rows live in its TMEM lane: no cross-thread reduction).
// Kernels: rf_attn_fa64_kernel (self-attention, 64-key tiles, double-buffered S) and
// rf_attn_fa_kernel (one 128-key tile: cross-attention when not fused into the cross-Q
// GEMM epilogue).
#include <stdlib.h>

#include "rf_common.cuh"
#include "rf_gemm_host.h"
#include "rf_sm100.cuh"

namespace rf {

using namespace rf::sm100;

constexpr int kTcRows = 128;                 // query rows per CTA = keys per tile = head dim
constexpr uint32_t kTile = 128 * 64 * 2;     // one SW128 K-major tile: 128 rows x 64 bf16
constexpr uint32_t kOperand = 2 * kTile;     // 128 x 128 bf16 operand (two K tiles)
// NH query heads per CTA sharing one KV head (GQA): Q[NH], K[2 stages], V[3 - NH stages], P[NH]
template <int NH>
constexpr size_t attn_smem() {
    return 1024 + (size_t)(NH + 2 + (3 - NH) + NH) * kOperand + 128;
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------------
// Single-pass attention with head ping-pong (the default).
//
// CTA = one 128-row query tile x NH query heads sharing a KV head.  Warps 0..4NH-1 run
// the softmax (warp w: head w / 4, TMEM lane quarter w % 4, one query row per thread);
// warp 4NH issues the MMAs (one elected thread), warp 4NH+1 issues the TMA loads.
// Per head a and key tile j:  S_a = Q_a K_j^T (SS MMA into TMEM) -> softmax threads read S,
// keep a running row max m with LAZY rescaling (O and l are rescaled only when the tile
// max exceeds m by more than 2^8, so P <= 256 stays exact in bf16/fp32), write
// P = exp2(S*scale - m) as bf16 into the same TMEM columns -> O_a += P V_j (TS MMA: A from
// TMEM, V^T from shared memory).  The MMA thread issues PV_a(j), then S_a(j+1), then the
// other head's pair, so head 1's softmax overlaps head 0's MMAs and vice versa.
// K and V^T are double-buffered; one pass over the keys (no recomputed S).
// TMEM: per head S/P 128 columns + O 128 columns (512 for NH = 2).
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// (x0, x1) * s + (c, c) with one packed FFMA2 (sm_100)
__device__ __forceinline__ float2 fma2(float2 x, float s, float c) {
    uint64_t r;
    asm("{\n.reg .b64 a, b, d;\n"
        "mov.b64 a, {%1, %2};\n"
        "mov.b64 b, {%3, %3};\n"
        "mov.b64 d, {%4, %4};\n"
        "fma.rn.ftz.f32x2 %0, a, b, d;\n}"
        : "=l"(r)
        : "f"(x.x), "f"(x.y), "f"(s), "f"(c));
    return make_float2(__uint_as_float((uint32_t)r), __uint_as_float((uint32_t)(r >> 32)));
}



// 2^x for a pair on the FMA pipe (x <= 8 or -inf): round-to-nearest split x = j + f with
// f in [-1/2, 1/2] (magic-number add), 2^f by a degree-3 polynomial (max rel. error 7.7e-5,
// far below P's bf16 step of 3.9e-3), j added to the exponent bits with one integer
// multiply-add.  The MUFU ex2 unit (16 / clk / SM) is the softmax's bottleneck; computing a
// share of the exponentials here balances the two pipes.
__device__ __forceinline__ uint64_t pk2(float a, float b) {
    return (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(b) << 32);
}
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
    constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23: x + kMagic rounds x to an integer
    const float x0 = fmaxf(x.x, -125.f), x1 = fmaxf(x.y, -125.f);
    uint64_t t, j, f, p;
    asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk2(x0, x1)), "l"(pk2(kMagic, kMagic)));
    asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(j) : "l"(t), "l"(pk2(kMagic, kMagic)));
    asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(f) : "l"(pk2(x0, x1)), "l"(j));
    asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(f), "l"(pk2(0.05508868f, 0.05508868f)),
        "l"(pk2(0.24260405f, 0.24260405f)));
    asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(f), "l"(p), "l"(pk2(0.69327624f, 0.69327624f)));
    asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(f), "l"(p), "l"(pk2(0.99992894f, 0.99992894f)));
    const uint32_t r0 = (uint32_t)t * (1u << 23) + (uint32_t)p;
    const uint32_t r1 = (uint32_t)(t >> 32) * (1u << 23) + (uint32_t)(p >> 32);
    return make_float2(__uint_as_float(r0), __uint_as_float(r1));
}

constexpr int kPolyPairs = 0;   // of 16 exponential pairs per 32-column chunk (see exp2_poly2)

// NH = 2: three full warpgroups (two softmax groups + one with the MMA and TMA warps) so
// registers can be moved between them with setmaxnreg; NH = 1: softmax group + 2 warps.
constexpr int fa_threads(int nh) { return nh == 2 ? 384 : 128 * nh + 64; }

template <int NH, int KVS>
constexpr size_t fa_smem() {
    return 1024 + (size_t)(NH + 2 * KVS) * kOperand + 256;
}

// debugging timeline ([cta][16 events][16] u64: clock64 per key tile j < 15, globaltimer / SM id in the
// last slots), set by rf_attn_set_trace; null in production
__device__ unsigned long long *g_attn_trace = nullptr;
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define FA_GTRACE(ev)                                                                                     \
    do {                                                                                                  \
        if (trace_buf)                                                                                    \
            trace_buf[((size_t)(blockIdx.y * gridDim.x + blockIdx.x) * 16 + (ev)) * 16 + 15] = globaltimer(); \
    } while (0)
#define FA_TRACE(ev, j)                                                                                  \
    do {                                                                                                 \
        if (trace_buf && (j) < 15)                                                                       \
            trace_buf[((size_t)(blockIdx.y * gridDim.x + blockIdx.x) * 16 + (ev)) * 16 + (j)] = clock64(); \
    } while (0)

// KVS = K/V stages: 2 (double-buffered) or 1 (one key tile, e.g. the cross-attention: the
// CTA then fits twice per SM -- NH = 1, KVS = 1: 96 KB shared memory, 256 TMEM columns).
// PE = exponential pairs (of every 16) computed by exp2_poly2 instead of MUFU ex2.
template <int NH, int KVS, int PE, bool PP>
__global__ void __launch_bounds__(fa_threads(NH), (NH == 1 && KVS == 1) ? 2 : 1)
rf_attn_fa_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                  const __grid_constant__ CUtensorMap tvt, __nv_bfloat16 *__restrict__ out, int64_t ldo, int Nq,
                  int Nk, int H, int Hkv, float scale_log2) {
    extern __shared__ uint8_t smem_raw[];
    unsigned long long *const trace_buf = g_attn_trace;   // debugging timeline (null in production)
    uint8_t *base = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sQ = base;                 // [NH]
    uint8_t *sK = sQ + NH * kOperand;     // [KVS]
    uint8_t *sV = sK + KVS * kOperand;    // [KVS] V^T tiles (rows = head dims, K-major over keys)
    uint64_t *bar = (uint64_t *)(sV + KVS * kOperand);
    uint64_t *qfull = bar, *kfull = bar + 1, *kempty = bar + 3, *vfull = bar + 5, *vempty = bar + 7;
    uint64_t *sfull = bar + 9, *pfull = bar + 11, *odone = bar + 13;
    uint32_t *tmem_slot = (uint32_t *)(bar + 16);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int MMA_WARP = 4 * NH, TMA_WARP = 4 * NH + 1;
    const int group = H / Hkv;
    const int bh = blockIdx.y, per_b = H / NH, b = bh / per_b, h0 = (bh % per_b) * NH;
    const int hk = h0 / group;
    const int q0 = blockIdx.x * kTcRows;
    const int nt = (Nk + kTcRows - 1) / kTcRows;
    constexpr uint32_t idesc = idesc_bf16(128, 128);

    if (tid == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        tma_prefetch(&tvt);
        mbar_init(qfull, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&kfull[i], 1);
            mbar_init(&kempty[i], 1);
            mbar_init(&vfull[i], 1);
            mbar_init(&vempty[i], 1);
            mbar_init(&sfull[i], 1);
            mbar_init(&pfull[i], 4);   // the 4 softmax warps of the head
            mbar_init(&odone[i], 1);
        }
        mbar_fence_init();
    }
    if (warp == MMA_WARP) tmem_alloc<256 * NH>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_launch();
    if (tid == 0) FA_GTRACE(0);
    // NH = 2: the softmax threads hold a whole 128-column S row in registers; setmaxnreg gives
    // them the registers the MMA / TMA warpgroup does not need (the CTA pool is 384 x 168 at launch: 8 x 200 + 4 x 96 warps fit)
    if (warp >= MMA_WARP) {
      if constexpr (NH == 2) asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
      if (warp == TMA_WARP) {
        if (elect_one()) {
            mbar_expect_tx(qfull, NH * kOperand);
            for (int a = 0; a < NH; ++a) {
                tma_load_2d(sQ + a * kOperand, &tq, qfull, (h0 + a) * 128, b * Nq + q0);
                tma_load_2d(sQ + a * kOperand + kTile, &tq, qfull, (h0 + a) * 128 + 64, b * Nq + q0);
            }
            for (int j = 0; j < nt; ++j) {
                const int s = j % KVS;
                const uint32_t ph = ((j / KVS) & 1) ^ 1;
                mbar_wait(&kempty[s], ph);
                mbar_expect_tx(&kfull[s], kOperand);
                tma_load_2d(sK + s * kOperand, &tk, &kfull[s], hk * 128, b * Nk + j * 128);
                tma_load_2d(sK + s * kOperand + kTile, &tk, &kfull[s], hk * 128 + 64, b * Nk + j * 128);
                mbar_wait(&vempty[s], ph);
                mbar_expect_tx(&vfull[s], kOperand);
                tma_load_2d(sV + s * kOperand, &tvt, &vfull[s], j * 128, (b * Hkv + hk) * 128);
                tma_load_2d(sV + s * kOperand + kTile, &tvt, &vfull[s], j * 128 + 64, (b * Hkv + hk) * 128);
            }
        }
      } else if (warp == MMA_WARP) {
        if (elect_one()) {
            auto mma_s = [&](int a, int s) {   // S_a = Q_a K_s^T
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t ad = sdesc_sw128(sQ + a * kOperand + (ks >> 2) * kTile) + (uint64_t)((ks & 3) * 2);
                    const uint64_t bd = sdesc_sw128(sK + s * kOperand + (ks >> 2) * kTile) + (uint64_t)((ks & 3) * 2);
                    umma_bf16(tmem + a * 128, ad, bd, idesc, ks > 0);
                }
                umma_commit(&sfull[a]);
            };
            auto mma_o = [&](int a, int s, bool acc) {   // O_a += P_a V_s (P_a in TMEM over S_a)
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t bd = sdesc_sw128(sV + s * kOperand + (ks >> 2) * kTile) + (uint64_t)((ks & 3) * 2);
                    umma_bf16_ts(tmem + NH * 128 + a * 128, tmem + a * 128 + ks * 8, bd, idesc,
                                 (acc || ks > 0) ? 1u : 0u);
                }
                umma_commit(&odone[a]);
            };
            mbar_wait(qfull, 0);
            mbar_wait(&kfull[0], 0);
            tc_fence_after();
            for (int a = 0; a < NH; ++a) mma_s(a, 0);
            umma_commit(&kempty[0]);
            for (int j = 0; j < nt; ++j) {
                const int s = j % KVS, s1 = (j + 1) % KVS;
                for (int a = 0; a < NH; ++a) {
                    mbar_wait(&pfull[a], j & 1);
                    if (a == 0) mbar_wait(&vfull[s], (j / KVS) & 1);
                    tc_fence_after();
                    FA_TRACE(a, j);
                    mma_o(a, s, j > 0);
                    if (a == NH - 1) umma_commit(&vempty[s]);
                    if (j + 1 < nt) {
                        // no wait for PV_a(j): tcgen05.mma executes in issue order, so S_a(j+1)
                        // cannot overwrite the P_a(j) columns before PV_a(j) has read them
                        if (a == 0) mbar_wait(&kfull[s1], ((j + 1) / KVS) & 1);
                        tc_fence_after();
                        FA_TRACE(2 + a, j + 1);
                        mma_s(a, s1);
                        if (a == NH - 1) umma_commit(&kempty[s1]);
                    }
                }
            }
        }
      }
    } else {
        if constexpr (NH == 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
        // softmax warps: thread owns query row `row` of head a
        const int a = warp >> 2, quarter = warp & 3;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        const uint32_t tS = tmem + lane_base + a * 128, tO = tmem + lane_base + NH * 128 + a * 128;
        float m = 0.f, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            mbar_wait(&sfull[a], j & 1);
            if constexpr (PP && NH == 2) {
                // strict ping-pong: head 1's softmax of tile j starts when head 0's has
                // finished, head 0's of tile j + 1 when head 1's of tile j has -- the two
                // softmax groups take turns on the exp/issue pipes while the tensor core
                // works for the other head
                if (a == 1) mbar_wait(&pfull[0], j & 1);
                else if (j > 0) mbar_wait(&pfull[1], (j - 1) & 1);
            }
            tc_fence_after();
            if (quarter == 0 && lane == 0) FA_TRACE(4 + a, j);
            const int valid = Nk - j * 128;
            uint32_t r[128];   // the whole S row of this thread (one TMEM pass)
            tmem_ld32(tS, *(uint32_t(*)[32])(r));
            tmem_ld32(tS + 32, *(uint32_t(*)[32])(r + 32));
            tmem_ld32(tS + 64, *(uint32_t(*)[32])(r + 64));
            tmem_ld32(tS + 96, *(uint32_t(*)[32])(r + 96));
            tmem_ld_wait();
            if (quarter == 0 && lane == 0) FA_TRACE(8 + a, j);
            if (valid < 128) {   // the last key tile: keys >= valid are masked
#pragma unroll
                for (int e = 0; e < 128; ++e)
                    if (e >= valid) r[e] = __float_as_uint(-INFINITY);
            }
            // row max as 4 independent 3-input max chains (a single chain is 64 dependent ops)
            float mx[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) mx[q] = fmaxf(__uint_as_float(r[q]), __uint_as_float(r[q + 4]));
#pragma unroll
            for (int e = 8; e < 128; e += 8)
#pragma unroll
                for (int q = 0; q < 4; ++q) mx[q] = fmaxf(mx[q], fmaxf(__uint_as_float(r[e + q]), __uint_as_float(r[e + q + 4])));
            float tmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
            tmax *= scale_log2;
            if (j == 0) {
                m = tmax;
            } else {
                const bool need = tmax > m + 8.f;
                if (__any_sync(0xffffffffu, need)) {   // lazy rescale of O and l (warp-uniform TMEM traffic)
                    const float mn = need ? tmax : m;
                    const float f = ex2_approx(m - mn);
                    l *= f;
                    m = mn;
#pragma unroll 1
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                        tmem_st32(tO + c * 32, o);
                    }
                    tmem_st_wait();
                }
            }
            // P = exp2(S * scale - m) as bf16 pairs into the first 64 columns of S (the row is
            // in registers).  Arguments are <= 8 (lazy max) or -inf (masked): the MUFU ex2
            // needs no range fix-up.  l sums the fp32 values (the bf16 rounding of P is below
            // the output's own bf16 step).
            const float nm = -m;
            if (quarter == 0 && lane == 0) FA_TRACE(10 + a, j);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t pk[16];
                uint64_t ls = 0;   // packed (even, odd) partial sums
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float2 x = fma2(make_float2(__uint_as_float(r[c * 32 + 2 * e]),
                                                      __uint_as_float(r[c * 32 + 2 * e + 1])),
                                          scale_log2, nm);
                    const float2 pv = e < PE ? exp2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
                    asm("add.rn.ftz.f32x2 %0, %0, %1;" : "+l"(ls) : "l"(pk2(pv.x, pv.y)));
                    __nv_bfloat162 hh = __floats2bfloat162_rn(pv.x, pv.y);
                    pk[e] = *(uint32_t *)&hh;
                }
                l += __uint_as_float((uint32_t)ls) + __uint_as_float((uint32_t)(ls >> 32));
                tmem_st16(tS + c * 16, pk);
            }
            if (quarter == 0 && lane == 0) FA_TRACE(12 + a, j);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull[a]);
            if (quarter == 0 && lane == 0) FA_TRACE(6 + a, j);
        }
        mbar_wait(&odone[a], (nt - 1) & 1);
        tc_fence_after();
        const float inv_l = l > 0.f ? 1.f / l : 0.f;
        const int qrow = q0 + quarter * 32 + lane;
        const int h = h0 + a;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + c * 32, r);
            tmem_ld_wait();
            uint4 pk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t *w = (uint32_t *)&pk[q];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(r[q * 8 + 2 * e]) * inv_l,
                                                              __uint_as_float(r[q * 8 + 2 * e + 1]) * inv_l);
                    w[e] = *(uint32_t *)&hh;
                }
            }
            // warp-collective: 8 query rows x 64 contiguous bytes per store (rows >= Nq skipped)
            store_rows_bf16x32(out + (int64_t)b * Nq * ldo, ldo, qrow - lane, Nq, h * 128 + c * 32, lane, pk);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) FA_GTRACE(1);
    if (warp == MMA_WARP) tmem_dealloc<256 * NH>(tmem);
}

// ---------------------------------------------------------------------------------
// Self-attention over 64-key tiles with double-buffered scores (the default when the GQA
// head pair shares a KV head and there is more than one 128-key tile).
//
// CTA = one 128-row query tile x NH query heads of one KV head: warpgroup a runs head a's
// softmax (one query row per thread), warp 4 NH issues the MMAs, warp 4 NH + 1 the TMA
// loads.  NH = 1 fits two CTAs per SM (96 KB shared memory, 256 TMEM columns): the two
// CTAs' softmax and MMA phases interleave, and 384 head tiles balance over 296 slots
// better than 192 head-pair tiles over 148.  Per head, S_j = Q K_j^T (M=128, N=64) goes into one of two
// 64-column TMEM buffers, so S_{j+1} is computed while the softmax works on S_j: the
// tensor core never waits for the softmax and the softmax never waits for a fresh S.
// P_j (bf16) overwrites the first 32 columns of its S buffer and O += P_j V_j reads it
// from TMEM (TS MMA, V^T tile K-major over keys).  MMA order per head:
// ... PV(j-1), S(j+1), PV(j), S(j+2) ... -- tcgen05 executes in issue order, so S(j+2)
// cannot overwrite P(j) before PV(j) has read it.  Running max with lazy O rescaling
// (only when the tile max grows by more than 2^8; the softmax first waits for PV(j-1)).
// TMEM: head a: S buffers at columns a*128 + {0, 64}, O at NH*128 + a*128.
// K / V^T tiles: KS-stage rings of 16 KB each (KS = 4 for NH = 2, 2 for NH = 1).
constexpr int kKeys64 = 64;
template <int NH>
constexpr int fa64_stages() { return NH == 2 ? 4 : 2; }
constexpr uint32_t kK64Half = 64 * 64 * 2;        // [64 keys][64 dims] bf16, SW128
constexpr uint32_t kK64Tile = 2 * kK64Half;       // [64 keys][128 dims]
constexpr uint32_t kV64Tile = 128 * 64 * 2;       // [128 dims][64 keys]
template <int NH>
constexpr size_t fa64_smem() {
    return 1024 + NH * (size_t)kOperand + fa64_stages<NH>() * (size_t)(kK64Tile + kV64Tile) + 256;
}

template <int NH, int PE>
__global__ void __launch_bounds__(128 * NH + 64, NH == 1 ? 2 : 1)
rf_attn_fa64_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tvt, __nv_bfloat16 *__restrict__ out, int64_t ldo, int Nq,
                    int Nk, int H, int Hkv, float scale_log2) {
    constexpr int KS = fa64_stages<NH>();
    extern __shared__ uint8_t smem_raw[];
    unsigned long long *const trace_buf = g_attn_trace;   // debugging timeline (null in production)
    uint8_t *base = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sQ = base;                    // [NH heads] x 32 KB
    uint8_t *sK = sQ + NH * kOperand;      // [KS] x 16 KB
    uint8_t *sV = sK + KS * kK64Tile;      // [KS] x 16 KB (V^T: rows = head dims)
    uint64_t *bar = (uint64_t *)(sV + KS * kV64Tile);
    uint64_t *qfull = bar, *kfull = bar + 1, *kempty = kfull + KS, *vfull = kempty + KS, *vempty = vfull + KS;
    uint64_t *sfull = vempty + KS;         // [head * 2 + buffer]
    // odone[head * 2 + (j & 1)]: PV(j) completion, alternating by tile parity so a waiter that
    // skipped phases still reads an unambiguous parity (see the rescale wait below).
    // pfull[head * 2 + (j & 1)]: P(j) written, alternating by tile parity too: the softmax can
    // finish tiles j AND j + 1 (S(j + 1) is issued before the MMA warp waits for P(j)) before
    // the MMA warp first polls, and one barrier would then be two phases ahead of its waiter,
    // whose parity wait can never succeed (a hang caught by the RF_HANG_TRAP build).  With a
    // barrier per parity, P(j + 2) -- which needs S(j + 2), issued only after the wait -- is
    // the earliest that could complete the waited barrier's next phase.
    uint64_t *pfull = sfull + 2 * NH, *odone = pfull + 2 * NH;
    uint32_t *tmem_slot = (uint32_t *)(odone + 2 * NH);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int MMA_WARP = 4 * NH, TMA_WARP = 4 * NH + 1;
    constexpr uint32_t TO = NH * 128;      // O column base in TMEM
    const int group = H / Hkv;
    const int bh = blockIdx.y, per_b = H / NH, b = bh / per_b, h0 = (bh % per_b) * NH;
    const int hk = h0 / group;
    const int q0 = blockIdx.x * kTcRows;
    const int nt = (Nk + kKeys64 - 1) / kKeys64;
    constexpr uint32_t idesc_s = idesc_bf16(128, 64), idesc_o = idesc_bf16(128, 128);

    if (tid == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        tma_prefetch(&tvt);
        mbar_init(qfull, 1);
        for (int i = 0; i < KS; ++i) {
            mbar_init(&kfull[i], 1);
            mbar_init(&kempty[i], 1);
            mbar_init(&vfull[i], 1);
            mbar_init(&vempty[i], 1);
        }
        for (int i = 0; i < 2 * NH; ++i) mbar_init(&sfull[i], 1);
        for (int i = 0; i < 2 * NH; ++i) mbar_init(&pfull[i], 4);   // the 4 softmax warps of the head
        for (int i = 0; i < 2 * NH; ++i) mbar_init(&odone[i], 1);
        mbar_fence_init();
    }
    if (warp == MMA_WARP) tmem_alloc<256 * NH>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_launch();
    if (tid == 0) {
        FA_GTRACE(0);
        // NH = 1 leaves event row 3 free: SM id, entry and exit clocks (tools/attn_trace.py)
        if (trace_buf) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            unsigned long long *r3 = trace_buf + ((size_t)(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 3) * 16;
            r3[15] = smid;
            r3[14] = clock64();
        }
    }

    if (warp == TMA_WARP) {
        if (elect_one()) {
            mbar_expect_tx(qfull, NH * kOperand);
            for (int a = 0; a < NH; ++a) {
                tma_load_2d(sQ + a * kOperand, &tq, qfull, (h0 + a) * 128, b * Nq + q0);
                tma_load_2d(sQ + a * kOperand + kTile, &tq, qfull, (h0 + a) * 128 + 64, b * Nq + q0);
            }
            for (int j = 0; j < nt; ++j) {
                const int s = j % KS;
                const uint32_t ph = ((j / KS) & 1) ^ 1;
                mbar_wait(&kempty[s], ph);
                FA_TRACE(13, j);
                mbar_expect_tx(&kfull[s], kK64Tile);
                tma_load_2d(sK + s * kK64Tile, &tk, &kfull[s], hk * 128, b * Nk + j * kKeys64);
                tma_load_2d(sK + s * kK64Tile + kK64Half, &tk, &kfull[s], hk * 128 + 64, b * Nk + j * kKeys64);
                mbar_wait(&vempty[s], ph);
                FA_TRACE(14, j);
                mbar_expect_tx(&vfull[s], kV64Tile);
                tma_load_2d(sV + s * kV64Tile, &tvt, &vfull[s], j * kKeys64, (b * Hkv + hk) * 128);
            }
        }
    } else if (warp == MMA_WARP) {
        if (elect_one()) {
            auto mma_s = [&](int a, int s, int buf) {   // S_a -> buffer buf
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t ad = sdesc_sw128(sQ + a * kOperand + (ks >> 2) * kTile) + (uint64_t)((ks & 3) * 2);
                    const uint64_t bd = sdesc_sw128(sK + s * kK64Tile + (ks >> 2) * kK64Half) + (uint64_t)((ks & 3) * 2);
                    umma_bf16(tmem + a * 128 + buf * 64, ad, bd, idesc_s, ks > 0);
                }
                umma_commit(&sfull[a * 2 + buf]);
            };
            auto mma_o = [&](int a, int s, int buf, bool acc) {   // O_a += P_a V (P in TMEM)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t bd = sdesc_sw128(sV + s * kV64Tile) + (uint64_t)(ks * 2);
                    umma_bf16_ts(tmem + TO + a * 128, tmem + a * 128 + buf * 64 + ks * 8, bd, idesc_o,
                                 (acc || ks > 0) ? 1u : 0u);
                }
                umma_commit(&odone[a * 2 + buf]);
            };
            mbar_wait(qfull, 0);
            for (int j = 0; j < 2 && j < nt; ++j) {
                mbar_wait(&kfull[j], 0);
                tc_fence_after();
                FA_TRACE(2, j);
#pragma unroll
                for (int a = 0; a < NH; ++a) mma_s(a, j, j);
                umma_commit(&kempty[j]);
            }
            for (int j = 0; j < nt; ++j) {
                const int s = j % KS, s2 = (j + 2) % KS, buf = j & 1;
#pragma unroll 1
                for (int a = 0; a < NH; ++a) {
                    mbar_wait(&pfull[a * 2 + (j & 1)], (j >> 1) & 1);
                    if (a == 0) mbar_wait(&vfull[s], (j / KS) & 1);
                    tc_fence_after();
                    FA_TRACE(a, j);
                    mma_o(a, s, buf, j > 0);
                    if (a == NH - 1) umma_commit(&vempty[s]);
                    if (j + 2 < nt) {
                        if (a == 0) mbar_wait(&kfull[s2], ((j + 2) / KS) & 1);
                        tc_fence_after();
                        FA_TRACE(2 + a, j + 2);
                        mma_s(a, s2, buf);
                        if (a == NH - 1) umma_commit(&kempty[s2]);
                    }
                }
            }
        }
    } else if (warp < MMA_WARP) {
        const int a = warp >> 2, quarter = warp & 3;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        const uint32_t tO = tmem + lane_base + TO + a * 128;
        float m = 0.f, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            const int buf = j & 1;
            const uint32_t tS = tmem + lane_base + a * 128 + buf * 64;
            mbar_wait(&sfull[a * 2 + buf], (j >> 1) & 1);
            tc_fence_after();
            if (quarter == 0 && lane == 0) FA_TRACE(4 + a, j);
            uint32_t r[64];
            tmem_ld32(tS, *(uint32_t(*)[32])(r));
            tmem_ld32(tS + 32, *(uint32_t(*)[32])(r + 32));
            tmem_ld_wait();
            if (quarter == 0 && lane == 0) FA_TRACE(8 + a, j);
            const int valid = Nk - j * kKeys64;
            if (valid < kKeys64) {   // the last key tile: keys >= valid are masked
#pragma unroll
                for (int e = 0; e < 64; ++e)
                    if (e >= valid) r[e] = __float_as_uint(-INFINITY);
            }
            float mx[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) mx[q] = fmaxf(__uint_as_float(r[q]), __uint_as_float(r[q + 4]));
#pragma unroll
            for (int e = 8; e < 64; e += 8)
#pragma unroll
                for (int q = 0; q < 4; ++q) mx[q] = fmaxf(mx[q], fmaxf(__uint_as_float(r[e + q]), __uint_as_float(r[e + q + 4])));
            const float tmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;
            if (j == 0) {
                m = tmax;
            } else {
                if (quarter == 0 && lane == 0) FA_TRACE(10 + a, j);
                const bool need = tmax > m + 8.f;
                if (__any_sync(0xffffffffu, need)) {   // lazy rescale of O and l
                    // O must be stable: wait for PV(j-1).  Its barrier also completes for PV(j-3),
                    // ..., all done (S(j)'s commit covers PV(j-2) and everything before), and PV(j+1)
                    // cannot have run: the barrier is on PV(j-1)'s phase or just past it.
                    mbar_wait(&odone[a * 2 + ((j - 1) & 1)], ((j - 1) >> 1) & 1);
                    tc_fence_after();
                    const float mn = need ? tmax : m;
                    const float f = ex2_approx(m - mn);
                    l *= f;
                    m = mn;
#pragma unroll 1
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                        tmem_st32(tO + c * 32, o);
                    }
                    tmem_st_wait();
                }
            }
            const float nm = -m;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t pk[16];
                uint64_t ls = 0;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float2 x = fma2(make_float2(__uint_as_float(r[c * 32 + 2 * e]),
                                                      __uint_as_float(r[c * 32 + 2 * e + 1])),
                                          scale_log2, nm);
                    const float2 pv = e < PE ? exp2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
                    asm("add.rn.ftz.f32x2 %0, %0, %1;" : "+l"(ls) : "l"(pk2(pv.x, pv.y)));
                    __nv_bfloat162 hh = __floats2bfloat162_rn(pv.x, pv.y);
                    pk[e] = *(uint32_t *)&hh;
                }
                l += __uint_as_float((uint32_t)ls) + __uint_as_float((uint32_t)(ls >> 32));
                tmem_st16(tS + c * 16, pk);
            }
            if (quarter == 0 && lane == 0) FA_TRACE(12 + a, j);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull[a * 2 + (j & 1)]);
            // keep the head's 4 warps within one tile of each other: pfull counts 4 arrivals per
            // phase, so a warp that raced ahead and arrived for tile j + 1 before a slow warp's
            // tile-j arrival would complete phase j early (PV(j) reading unfinished P rows)
            asm volatile("bar.sync %0, 128;" ::"r"(1 + a) : "memory");
            if (quarter == 0 && lane == 0) FA_TRACE(6 + a, j);
        }
        if (nt >= 2) mbar_wait(&odone[a * 2 + ((nt - 2) & 1)], ((nt - 2) >> 1) & 1);
        mbar_wait(&odone[a * 2 + ((nt - 1) & 1)], ((nt - 1) >> 1) & 1);
        tc_fence_after();
        const float inv_l = l > 0.f ? 1.f / l : 0.f;
        const int qrow = q0 + quarter * 32 + lane;
        const int h = h0 + a;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + c * 32, r);
            tmem_ld_wait();
            uint4 pk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t *w = (uint32_t *)&pk[q];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(r[q * 8 + 2 * e]) * inv_l,
                                                              __uint_as_float(r[q * 8 + 2 * e + 1]) * inv_l);
                    w[e] = *(uint32_t *)&hh;
                }
            }
            // warp-collective: 8 query rows x 64 contiguous bytes per store (rows >= Nq skipped)
            store_rows_bf16x32(out + (int64_t)b * Nq * ldo, ldo, qrow - lane, Nq, h * 128 + c * 32, lane, pk);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        FA_GTRACE(1);
        if (trace_buf) trace_buf[((size_t)(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 3) * 16 + 13] = clock64();
    }
    if (warp == MMA_WARP) tmem_dealloc<256 * NH>(tmem);
}

int attn_plan(AttnPlan *p, const void *q, int64_t ldq, int64_t q_cols, const void *k, int64_t ldk, int64_t k_cols,
              const void *vt, int B, int Nq, int Nk, int Nk_pad, int H, int Hkv) {
    if (H % Hkv || Nk_pad % 8 || Nk > Nk_pad) {
        set_error("attn_plan: bad shape");
        return RF_EINVAL;
    }
    int rc = make_tmap_bf16_2d(&p->tq, q, (uint64_t)q_cols, (uint64_t)B * Nq, (uint64_t)ldq * 2, 64, 128);
    if (!rc) rc = make_tmap_bf16_2d(&p->tk, k, (uint64_t)k_cols, (uint64_t)B * Nk, (uint64_t)ldk * 2, 64, 128);
    if (!rc)
        rc = make_tmap_bf16_2d(&p->tvt, vt, (uint64_t)Nk_pad, (uint64_t)B * Hkv * 128, (uint64_t)Nk_pad * 2, 64, 128);
    if (!rc) rc = make_tmap_bf16_2d(&p->tk64, k, (uint64_t)k_cols, (uint64_t)B * Nk, (uint64_t)ldk * 2, 64, 64);
    if (!rc)
        rc = make_tmap_bf16_2d(&p->tvt64, vt, (uint64_t)Nk_pad, (uint64_t)B * Hkv * 128, (uint64_t)Nk_pad * 2, 64, 64);
    p->B = B;
    p->Nq = Nq;
    p->Nk = Nk;
    p->Nk_pad = Nk_pad;
    p->H = H;
    p->Hkv = Hkv;
    return rc;
}

template <int NH, int KVS>
static int launch_fa(const AttnPlan &p, void *out, int64_t ldo, int B, float sc, cudaStream_t st) {
    constexpr bool PP = NH == 2;   // the GQA head pair ping-pongs its softmax groups
    static bool attr = false;
    if (!attr) {
        RF_TRY_CUDA(cudaFuncSetAttribute(rf_attn_fa_kernel<NH, KVS, kPolyPairs, PP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fa_smem<NH, KVS>()));
        attr = true;
    }
    dim3 grid((p.Nq + kTcRows - 1) / kTcRows, B * p.H / NH);
    RF_TRY_CUDA(launch_pdl(rf_attn_fa_kernel<NH, KVS, kPolyPairs, PP>, grid, dim3(fa_threads(NH)), fa_smem<NH, KVS>(),
                           st, p.tq, p.tk, p.tvt, (__nv_bfloat16 *)out, ldo, p.Nq, p.Nk, p.H, p.Hkv, sc));
    RF_TRY_LAUNCH("rf_attn_fa_kernel");
    return RF_OK;
}

template <int NH>
static int launch_fa64(const AttnPlan &p, void *out, int64_t ldo, int B, float sc, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        RF_TRY_CUDA(cudaFuncSetAttribute(rf_attn_fa64_kernel<NH, kPolyPairs>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)fa64_smem<NH>()));
        attr = true;
    }
    dim3 grid((p.Nq + kTcRows - 1) / kTcRows, B * p.H / NH);
    RF_TRY_CUDA(launch_pdl(rf_attn_fa64_kernel<NH, kPolyPairs>, grid, dim3(128 * NH + 64), fa64_smem<NH>(), st, p.tq,
                           p.tk64, p.tvt, (__nv_bfloat16 *)out, ldo, p.Nq, p.Nk, p.H, p.Hkv, sc));
    RF_TRY_LAUNCH("rf_attn_fa64_kernel");
    return RF_OK;
}

// Kernel choice for > 128 keys (development A/B through rf_attention_tc_bf16_kernel only;
// the DiT forward always takes the default).
static int g_self_kernel = 0;

int attn_run(const AttnPlan &p, void *out, int64_t ldo, int B, cudaStream_t st) {
    const float sc = 1.4426950408889634f / sqrtf(128.f);
    // one key tile (cross-attention to <= 128 conditioning tokens): one head per CTA, two
    // CTAs per SM; longer key ranges: 64-key tiles with double-buffered scores, one head per
    // CTA, two CTAs per SM (a 128-key-tile single-buffered variant measured slower: 33.2 vs
    // 31.1 us at config 2, 289 vs 269 us at 3000 tokens; profiles/r2_attention.txt)
    if (p.Nk <= kTcRows) return launch_fa<1, 1>(p, out, ldo, B, sc, st);
    switch (g_self_kernel) {
        default: return launch_fa64<1>(p, out, ldo, B, sc, st);
    }
}

}  // namespace rf

using namespace rf;

// Debugging aid (not part of the product ABI): per-CTA clock64 timeline of the single-pass
// attention ([cta][8 events][16 tiles] u64) -- see tools/attn_trace.py.
extern "C" int rf_attn_set_trace(void *buf) {
    unsigned long long *p = (unsigned long long *)buf;
    return cudaMemcpyToSymbol(g_attn_trace, &p, sizeof(p)) == cudaSuccess ? RF_OK : RF_ECUDA;
}

// Development entry (not used by the forward): the same attention with the kernel for > 128
// keys chosen explicitly (0 = the forward's default).
extern "C" int rf_attention_tc_bf16_kernel(int32_t kernel, const void *q, const void *k, const void *vt, void *out,
                                           int32_t batch, int32_t n_q, int32_t n_k, int32_t n_k_pad, int32_t heads,
                                           int32_t kv_heads, int64_t ldq, int64_t ldk, int64_t ldo, void *stream) {
    if (!q || !k || !vt || !out || batch < 1 || n_q < 1 || n_k < 1 || heads < 1 || kv_heads < 1 || kernel < 0 ||
        kernel > 1) {
        set_error("rf_attention_tc_bf16_kernel: bad arguments");
        return RF_EINVAL;
    }
    AttnPlan p;
    int rc = attn_plan(&p, q, ldq, (int64_t)heads * 128, k, ldk, (int64_t)kv_heads * 128, vt, batch, n_q, n_k,
                       n_k_pad, heads, kv_heads);
    if (rc) return rc;
    const int keep = g_self_kernel;
    g_self_kernel = kernel;
    rc = attn_run(p, out, ldo, batch, (cudaStream_t)stream);
    g_self_kernel = keep;
    return rc;
}

extern "C" int rf_attention_tc_bf16(const void *q, const void *k, const void *vt, void *out, int32_t batch,
                                    int32_t n_q, int32_t n_k, int32_t n_k_pad, int32_t heads, int32_t kv_heads,
                                    int64_t ldq, int64_t ldk, int64_t ldo, void *stream) {
    if (!q || !k || !vt || !out || batch < 1 || n_q < 1 || n_k < 1 || heads < 1 || kv_heads < 1) {
        set_error("rf_attention_tc_bf16: bad arguments");
        return RF_EINVAL;
    }
    AttnPlan p;
    int rc = attn_plan(&p, q, ldq, (int64_t)heads * 128, k, ldk, (int64_t)kv_heads * 128, vt, batch, n_q, n_k,
                       n_k_pad, heads, kv_heads);
    if (rc) return rc;
    return attn_run(p, out, ldo, batch, (cudaStream_t)stream);
}
