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
#include "rf_common.cuh"
#include "rf_sm100.cuh"

namespace rf::gemm {
using ::rf::pdl_wait;
using ::rf::pdl_launch;

enum Epi : int {
    kStoreBF16 = 0,   // out(bf16)[m,n] = acc
    kStoreF32 = 1,    // out(f32)[m,n] = acc
    kResidGate = 2,   // out(f32)[m,n] += gate[m / rows_per_batch, n] * acc   (AdaLN gated residual)
    kSwiGLU = 3,      // columns interleaved (g, u): out(bf16)[m, n/2] = silu(g) * u
    kStoreF32Scale = 4,  // out(f32)[m,n] = alpha * acc
    kBF16Rope = 5,    // out(bf16)[m,n] = acc, interleaved-pair RoPE on columns < rope_cols
    kCrossAttn = 6,   // acc = one 128-column query head of 128 rows -> cross-attention in the
                      // epilogue: out(bf16)[m, head cols] = softmax(q K_b^T / sqrt(128)) V_b
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
    // With vt_period > 0 the columns repeat in groups of vt_period (one group per layer of
    // a batched all-layer projection): within-group column c = n % vt_period, group
    // g = n / vt_period, and group g's V^T block starts vt_layer_stride elements later.
    __nv_bfloat16 *vt;
    int vt_col0, vt_heads;
    int64_t vt_ld;
    int vt_period;
    int64_t vt_layer_stride;
    // debugging: per-CTA clock64 timeline ([cta][tile < 16][8]); null in production
    unsigned long long *trace;
    // RMSNorm fused across a GEMM boundary (the norm without modulation before the
    // cross-attention query projection):
    //  kResidGate (TMA-staged): with aux set, also aux[m * aux_ld + n] = bf16 of the
    //    updated residual and sq_part[(n / 128) * sq_ld + m] = its sum of squares over
    //    each 128 columns (ascending column order, whatever BN);
    //  kStoreBF16: with rs_part set, acc is scaled by rsqrt(sum_t rs_part[t * rs_ld + m] *
    //    rs_inv_d + rs_eps) (t ascending) before rounding -- the consumer applies the norm.
    __nv_bfloat16 *aux;
    int64_t aux_ld;
    float *sq_part;
    int64_t sq_ld;
    const float *rs_part;
    int64_t rs_ld;
    int rs_tiles;
    float rs_inv_d, rs_eps;
    // kCrossAttn: rows are tiled per batch entry (x_rpb rows each, x_mtpb tiles of 128), so a
    // tile's rows all attend to the same batch entry's x_nk keys (K via tma_k, V^T via tma_vt,
    // the attention kernel's maps); query head = n / 128, KV head = head / x_group.
    int x_rpb, x_mtpb, x_batches, x_nk, x_group, x_hkv;
    float x_scale;   // log2(e) / sqrt(head dim)
    // B is constant across kernels (model weights): the producer may request its first
    // weight blocks before griddepcontrol.wait
    int b_static;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// globaltimer (ns) stamps: kernel entry -> [cta][15][7], exit -> [cta][14][7]
#define RF_GTRACE(tile)                                                                          \
    do {                                                                                         \
        if (epi.trace && threadIdx.x == 0) epi.trace[((size_t)blockIdx.x * 16 + (tile)) * 8 + 7] = gtimer(); \
    } while (0)

#define RF_TRACE(tile, slot)                                                                          \
    do {                                                                                              \
        if (epi.trace && (tile) < 16)                                                                 \
            epi.trace[((size_t)blockIdx.x * 16 + (tile)) * 8 + (slot)] = (unsigned long long)clock64(); \
    } while (0)

constexpr int BM = 128, BK = 64;
// CG = 1: one CTA per 128 x BN tile.  CG = 2: a CTA pair ((2,1,1) cluster) per 256 x BN
// tile -- each CTA stages its own 128 A rows and BN/2 of the B rows, the even CTA issues
// tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' shared memory, and each CTA's
// TMEM receives its own 128 accumulator rows.  Per-SM shared-memory operand traffic per
// FLOP drops by a third (BN = 256) to a quarter (BN = 128).
// TMA_C (the gated-residual epilogue at BN = 128): each epilogue warp prefetches its 32 x BN
// fp32 slice of the residual stream into shared memory with TMA (issued before the
// accumulator is ready, so the read overlaps the main loop), updates it in place from TMEM,
// and writes it back with a TMA store -- instead of row-per-thread global loads/stores.
// CC: residual columns staged per pass (BN: one pass per tile; 64: two passes, half the
// staging memory, two more operand stages -- for long K, where the main loop hides the
// epilogue anyway and latency tolerance matters more).
template <int BN, int CG = 1, int EPI = 0, int CC = BN>
struct Cfg {
    static constexpr int BN_LOAD = BN / CG;   // B rows staged by each CTA
    static constexpr uint32_t A_BYTES = BM * BK * 2;
    static constexpr uint32_t B_BYTES = BN_LOAD * BK * 2;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr bool TMA_C = EPI == 2;
    static constexpr bool XATT = EPI == 6;   // Q, K, V^T staging (32 KB each) for the epilogue attention
    // TMA_O (SwiGLU, BN = 256): each epilogue warp stages its [32 rows][128 cols] bf16 output
    // in shared memory (two SWIZZLE_128B boxes of 64 columns) and writes it with TMA stores:
    // full-line writes instead of one 16-byte store per row per thread
    static constexpr bool TMA_O = EPI == 3 && BN == 256;
    static constexpr int C_COLS = CC;                                           // staged per pass
    static constexpr uint32_t C_WARP_BYTES = TMA_C ? 32u * C_COLS * 4u : (TMA_O ? 32u * 128u * 2u : 0u);
    static constexpr uint32_t GATE_WARP_BYTES = TMA_C ? 2u * BN * 4u : 0u;   // the two gate rows a warp can touch
    static constexpr uint32_t C_BYTES = 4 * C_WARP_BYTES + 4 * GATE_WARP_BYTES + (XATT ? (CG == 1 ? 3u * 32768u : 65536u) : 0u);
    // as many operand stages as fit next to the epilogue staging (227 KB opt-in limit)
    static constexpr uint32_t BUDGET = 232448u - 1024u - 512u - C_BYTES;
    static constexpr int STAGES = (int)(BUDGET / STAGE_BYTES) > 10 ? 10 : (int)(BUDGET / STAGE_BYTES);
    static constexpr size_t SMEM = 1024 + STAGES * STAGE_BYTES + C_BYTES + 512;
};

__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16(x)); }
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *(uint32_t *)&h;
}

template <int BN, int EPI, int CG = 1, int CC = BN>
__global__ void __launch_bounds__(192, 1)
rf_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
               const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ CUtensorMap tma_k,
               const __grid_constant__ CUtensorMap tma_vt, int M, int N, int K, EpiArgs epi) {
    using namespace rf::sm100;
    using C = Cfg<BN, CG, EPI, CC>;
    constexpr int TM = BM * CG;   // output rows per tile (per CTA pair when CG = 2)
    constexpr int STAGES = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = base;
    uint8_t *sB = base + STAGES * C::A_BYTES;
    uint8_t *sC = sB + STAGES * C::B_BYTES;   // C_BYTES (1024-aligned: stage sizes are multiples of 1 KB)
    uint64_t *full = (uint64_t *)(sC + C::C_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint64_t *cfull = tempty + 2;            // [4] one per epilogue warp (TMA_C)
    uint64_t *xbar = cfull + 4;              // [5] kCrossAttn: K/V loaded, S done, O done, Q ready, P ready
    uint32_t *tmem_slot = (uint32_t *)(xbar + 5);
    static_assert(!C::XATT || BN == 128, "cross-attention epilogue: 128-wide tiles (one query head)");
    constexpr uint32_t TMEM_COLS = C::XATT ? 512 : 2 * BN;   // + S and O of the epilogue attention

    RF_GTRACE(15);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;   // 0 = leader (issues the MMAs)
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        if constexpr (C::TMA_C || C::TMA_O) tma_prefetch(&tma_c);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4 * CG);   // the epilogue warps of both CTAs release the leader
        }
        for (int i = 0; i < 4; ++i) mbar_init(&cfull[i], 1);
        for (int i = 0; i < 3; ++i) mbar_init(&xbar[i], 1);
        for (int i = 3; i < 5; ++i) mbar_init(&xbar[i], CG);   // one arrival per CTA of the pair
        if constexpr (C::XATT) {
            tma_prefetch(&tma_k);
            tma_prefetch(&tma_vt);
        }
        mbar_fence_init();
    }
    if (warp == 1) {
        if constexpr (CG == 2)
            tmem_alloc_pair<TMEM_COLS>(tmem_slot);
        else
            tmem_alloc<TMEM_COLS>(tmem_slot);
    }
    tc_fence_before();
    if constexpr (CG == 2)
        cluster_sync();   // peer barriers initialised before any remote arrive / complete_tx
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the previous kernel's outputs (A, the residual stream) are visible after pdl_wait; the
    // producer waits only after requesting the weight blocks of its first tile (below)
    if (warp != 0) pdl_wait();
    pdl_launch();
    RF_GTRACE(13);

    const int num_m = C::XATT ? epi.x_batches * epi.x_mtpb : (M + TM - 1) / TM, num_n = N / BN, kblocks = K / BK;
    // first row of tile t (kCrossAttn: tiles never straddle two batch entries)
    auto row0 = [&](int t) {
        const int mt = t % num_m;
        if constexpr (C::XATT) return (mt / epi.x_mtpb) * epi.x_rpb + (mt % epi.x_mtpb) * TM + (int)rank * BM;
        return mt * TM + (int)rank * BM;
    };
    const int num_tiles = num_m * num_n;
    const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;   // tile walker id
    const int units = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    // static tile walk: unit u takes tiles u, u + units, ... (every role walks the same
    // sequence); tiles whose rows lie beyond this call's M are skipped
    struct Walk {
        int pos;
    };
    auto walk_init = [&]() -> Walk { return Walk{unit}; };
    auto walk_next = [&](Walk &w, int &tile, int &kb0, int &kb1) -> bool {
        for (;;) {
            if (w.pos >= num_tiles) return false;
            tile = w.pos;
            kb0 = 0;
            kb1 = kblocks;
            w.pos += units;
            if (C::XATT || (tile % num_m) * TM < M) return true;
        }
    };

    if (warp == 0) {
        if (elect_one()) {
            // weights (B) stream through L2 once per forward: evict them first, so the
            // activations the next kernels read stay resident
            const uint64_t pol_w = createpolicy_evict_first();
            // The weights do not depend on the previous kernel: the first tile's first STAGES
            // weight blocks are requested before griddepcontrol.wait (a CTA that starts on an SM
            // the previous grid has left overlaps their DRAM latency with that grid's tail).
            // Fresh barriers: these stages' first empty waits would pass at once.
            int pre = 0;
            {
                int t, kb0, kb1;
                Walk w = walk_init();
                if (epi.b_static && walk_next(w, t, kb0, kb1)) {
                    const int n0 = (t / num_m) * BN + (int)rank * C::BN_LOAD;
                    pre = kb1 - kb0 < STAGES ? kb1 - kb0 : STAGES;
                    for (int s = 0; s < pre; ++s) {
                        if constexpr (CG == 2) {
                            if (rank == 0) mbar_expect_tx(&full[s], 2 * C::STAGE_BYTES);
                            tma_load_2d_pair_hint(sB + s * C::B_BYTES, &tma_b, mapa_shared(&full[s], 0), (kb0 + s) * BK,
                                                  n0, pol_w);
                        } else {
                            mbar_expect_tx(&full[s], C::STAGE_BYTES);
                            tma_load_2d_hint(sB + s * C::B_BYTES, &tma_b, &full[s], (kb0 + s) * BK, n0, pol_w);
                        }
                    }
                }
            }
            pdl_wait();
            int stage = 0;
            uint32_t phase = 0;
            int it = 0, t, kb0, kb1;
            for (Walk w = walk_init(); walk_next(w, t, kb0, kb1); ++it) {
                const int m0 = row0(t), n0 = (t / num_m) * BN + (int)rank * C::BN_LOAD;
                RF_TRACE(it, 6);
                for (int kb = kb0; kb < kb1; ++kb) {
                    const bool early = it == 0 && kb - kb0 < pre;   // B requested before pdl_wait
                    if (!early) mbar_wait(&empty[stage], phase ^ 1);
                    if constexpr (CG == 2) {
                        // both CTAs' bytes complete on the leader's full barrier
                        if (rank == 0 && !early) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
                        const uint32_t fb = mapa_shared(&full[stage], 0);
                        tma_load_2d_pair(sA + stage * C::A_BYTES, &tma_a, fb, kb * BK, m0);
                        if (!early) tma_load_2d_pair_hint(sB + stage * C::B_BYTES, &tma_b, fb, kb * BK, n0, pol_w);
                    } else {
                        if (!early) mbar_expect_tx(&full[stage], C::STAGE_BYTES);
                        tma_load_2d(sA + stage * C::A_BYTES, &tma_a, &full[stage], kb * BK, m0);
                        if (!early) tma_load_2d_hint(sB + stage * C::B_BYTES, &tma_b, &full[stage], kb * BK, n0, pol_w);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && elect_one()) {
            constexpr uint32_t idesc = idesc_bf16(TM, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            int it = 0, t, kb0, kb1;
            for (Walk w = walk_init(); walk_next(w, t, kb0, kb1); ++it) {
                RF_TRACE(it, 0);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                RF_TRACE(it, 1);
                const uint32_t d_tmem = tmem + acc * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (kb == kb0) RF_TRACE(it, 2);
                    const uint64_t ad = sdesc_sw128(sA + stage * C::A_BYTES);
                    const uint64_t bd = sdesc_sw128(sB + stage * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        if constexpr (CG == 2)
                            umma_bf16_pair(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc,
                                           (kb != kb0) || k != 0);
                        else
                            umma_bf16(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc,
                                      (kb != kb0) || k != 0);
                    }
                    if constexpr (CG == 2)
                        umma_commit_pair(&empty[stage]);
                    else
                        umma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                RF_TRACE(it, 3);
                if constexpr (CG == 2)
                    umma_commit_pair(&tfull[acc]);
                else
                    umma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if constexpr (C::TMA_C) {
        // gated residual, TMA-staged: out[m, n] += gate[m / rows_per_batch, n] * acc.  Each
        // epilogue warp owns a [32 rows][CC] fp32 slice of the residual stream in shared
        // memory per pass: loaded by TMA while the main loop runs (the next pass's slice is
        // requested as soon as the previous store has read the buffer), updated in place
        // from TMEM, written back with one TMA store per 32-column box.  The two gate rows
        // a 32-row slice can touch are staged in shared memory before the accumulator is
        // ready, and the accumulator is released before the last store.
        const int q = warp & 3;
        uint8_t *sw = sC + q * C::C_WARP_BYTES;   // NB boxes of [32 rows][32 fp32], SWIZZLE_128B
        float *gs = (float *)(sC + 4 * C::C_WARP_BYTES + q * C::GATE_WARP_BYTES);   // [2][BN] gate rows
        constexpr int NB = CC / 32, NP = BN / CC;
        static_assert((BN == 128 || BN == 256) && NB * 32 * NP == BN, "residual epilogue shape");
        auto tile_m0 = [&](int t) { return (t % num_m) * TM + (int)rank * BM + q * 32; };
        auto tile_n0 = [&](int t) { return (t / num_m) * BN; };
        auto load_pass = [&](int t, int p) {
            mbar_expect_tx(&cfull[q], C::C_WARP_BYTES);
#pragma unroll
            for (int j = 0; j < NB; ++j)
                tma_load_2d(sw + j * 4096, &tma_c, &cfull[q], tile_n0(t) + p * CC + j * 32, tile_m0(t));
        };
        int acc = 0, it = 0, t, kb0, kb1;
        uint32_t acc_phase = 0, c_phase = 0;
        Walk w = walk_init();
        bool have = walk_next(w, t, kb0, kb1);
        if (lane == 0 && have) load_pass(t, 0);
        while (have) {
            Walk wn = w;
            int tn, nk0, nk1;
            const bool next = walk_next(wn, tn, nk0, nk1);
            const bool next_load = next;
            const int m0 = tile_m0(t), n0 = tile_n0(t);
            {
            const int m = min(m0 + lane, M - 1);
            const int b_lo = min(m0, M - 1) / epi.rows_per_batch, b_hi = min(m0 + 31, M - 1) / epi.rows_per_batch;
            __syncwarp();   // the previous tile's gate reads are done
#pragma unroll
            for (int i = lane; i < BN / 4; i += 32) {
                ((float4 *)gs)[i] = __ldg((const float4 *)(epi.gate + (int64_t)b_lo * epi.gate_ld + n0) + i);
                ((float4 *)gs)[BN / 4 + i] = __ldg((const float4 *)(epi.gate + (int64_t)b_hi * epi.gate_ld + n0) + i);
            }
            __syncwarp();
            const float *gr = gs + (m / epi.rows_per_batch != b_lo ? BN : 0);
            const bool live = m0 + lane < M;
            float ss = 0.f;
            uint2 aux4[8];
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (q == 2 && lane == 0) RF_TRACE(it, 4);
#pragma unroll 1
            for (int p = 0; p < NP; ++p) {
                mbar_wait(&cfull[q], c_phase);
                c_phase ^= 1;
#pragma unroll 1
                for (int j = 0; j < NB; ++j) {
                    const int col = p * CC + j * 32;
                    uint32_t r[32];
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + col), r);
                    tmem_ld_wait();
                    float4 *row = (float4 *)(sw + j * 4096 + lane * 128);
                    const float4 *gv = (const float4 *)(gr + col);
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        const float4 g4 = gv[v];
                        float4 x = row[v ^ (lane & 7)];
                        x.x += g4.x * __uint_as_float(r[4 * v]);
                        x.y += g4.y * __uint_as_float(r[4 * v + 1]);
                        x.z += g4.z * __uint_as_float(r[4 * v + 2]);
                        x.w += g4.w * __uint_as_float(r[4 * v + 3]);
                        row[v ^ (lane & 7)] = x;
                        if (epi.aux) {   // the next RMSNorm's input (bf16) and its partial sum
                            ss = fmaf(x.x, x.x, ss);
                            ss = fmaf(x.y, x.y, ss);
                            ss = fmaf(x.z, x.z, ss);
                            ss = fmaf(x.w, x.w, ss);
                            aux4[v] = make_uint2(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w));
                        }
                    }
                    if (epi.aux) {   // warp-collective row stores (m0 = this warp's first row)
                        uint4 pk[4];
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            pk[v] = make_uint4(aux4[2 * v].x, aux4[2 * v].y, aux4[2 * v + 1].x, aux4[2 * v + 1].y);
                        store_rows_bf16x32(epi.aux, epi.aux_ld, m0, M, n0 + col, lane, pk);
                        // one partial sum of squares per 128 columns whatever the tile width, so
                        // the consumer's sum (and the row's result) does not depend on BN
                        if ((col + 32) % 128 == 0) {
                            if (live) epi.sq_part[(int64_t)((n0 + col) / 128) * epi.sq_ld + m0 + lane] = ss;
                            ss = 0.f;
                        }
                    }
                }
                if (p == NP - 1) tc_fence_before();
                fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the TMA store
                __syncwarp();
                if (lane == 0) {
                    if (p == NP - 1) {   // the accumulator has been read: release it
                        if constexpr (CG == 2)
                            mbar_arrive_cluster(mapa_shared(&tempty[acc], 0));
                        else
                            mbar_arrive(&tempty[acc]);
                    }
#pragma unroll
                    for (int j = 0; j < NB; ++j) tma_store_2d(&tma_c, sw + j * 4096, n0 + p * CC + j * 32, m0);
                    bulk_commit();
                    if (p == NP - 1 && q == 2) RF_TRACE(it, 5);
                    const bool more = p + 1 < NP || next_load;
                    if (more) {
                        bulk_wait_read0();   // the store has read the slice: the buffer is free
                        if (p + 1 < NP)
                            load_pass(t, p + 1);
                        else
                            load_pass(tn, 0);
                    }
                }
            }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
            w = wn;
            t = tn;
            kb0 = nk0;
            kb1 = nk1;
            have = next;
            ++it;
        }
        if (lane == 0) bulk_wait0();
    } else if constexpr (C::XATT) {
        // Cross-attention in the epilogue of the query projection.  Per tile (TM rows of one
        // batch entry x one query head): Q (accumulator, fused-norm scaled) -> bf16 SW128 tile
        // in smem; S = Q K^T (issued by one epilogue thread into TMEM columns 256..383 while
        // the MMA warp already runs the next tile's main loop); row softmax (one row per
        // thread, a single key tile: no rescaling); P (bf16) over S in TMEM; O = P V (TS MMA
        // into columns 384..511); O / l -> bf16 att.  K and V^T of the next tile are
        // prefetched by TMA as soon as this tile's MMAs have read them.
        // CG = 2 (CTA pairs, 256-row tiles): the attention MMAs are cta_group::2 as well, M =
        // 256 over both CTAs' Q / P rows; each CTA stages half of K (64 keys) and half of V^T
        // (64 dims), the leader CTA's thread issues S and PV once both CTAs' Q (P) are ready
        // (xq / xp count one arrival per CTA), and the commits multicast to both CTAs.
        const int q = warp & 3;
        const int row = q * 32 + lane;                       // row within this CTA's 128
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        constexpr uint32_t KV_HALF = CG == 1 ? 16384u : 8192u;   // one 64-dim (64-key) SW128 half
        uint8_t *sQ = sC, *sK = sC + 32768, *sV = sC + 32768 + 2 * KV_HALF;
        uint64_t *xk = xbar, *xs = xbar + 1, *xo = xbar + 2, *xq = xbar + 3, *xp = xbar + 4;
        const bool leader = q == 0 && lane == 0;                 // per CTA
        const bool issuer = leader && rank == 0;                 // issues the attention MMAs
        constexpr uint32_t idS = idesc_bf16(TM, 128);
        auto load_kv = [&](int t) {
            const int mt = t % num_m, b = mt / epi.x_mtpb, hk = (t / num_m) / epi.x_group;
            if constexpr (CG == 1) {
                mbar_expect_tx(xk, 65536);
                tma_load_2d(sK, &tma_k, xk, hk * 128, b * epi.x_nk);
                tma_load_2d(sK + 16384, &tma_k, xk, hk * 128 + 64, b * epi.x_nk);
                tma_load_2d(sV, &tma_vt, xk, 0, (b * epi.x_hkv + hk) * 128);
                tma_load_2d(sV + 16384, &tma_vt, xk, 64, (b * epi.x_hkv + hk) * 128);
            } else {   // this CTA's 64 keys of K and 64 dims of V^T (maps with 64 x 64 boxes)
                if (rank == 0) mbar_expect_tx(xk, 2 * 4 * KV_HALF);
                const uint32_t fb = mapa_shared(xk, 0);
                tma_load_2d_pair(sK, &tma_k, fb, hk * 128, b * epi.x_nk + (int)rank * 64);
                tma_load_2d_pair(sK + KV_HALF, &tma_k, fb, hk * 128 + 64, b * epi.x_nk + (int)rank * 64);
                tma_load_2d_pair(sV, &tma_vt, fb, 0, (b * epi.x_hkv + hk) * 128 + (int)rank * 64);
                tma_load_2d_pair(sV + KV_HALF, &tma_vt, fb, 64, (b * epi.x_hkv + hk) * 128 + (int)rank * 64);
            }
        };
        auto arrive_leader = [&](uint64_t *bar) {   // one arrival per CTA on the leader's barrier
            if constexpr (CG == 2)
                mbar_arrive_cluster(mapa_shared(bar, 0));
            else
                mbar_arrive(bar);
        };
        auto epi_sync = [] { asm volatile("bar.sync 1, 128;" ::: "memory"); };
        int acc = 0, it = 0;
        uint32_t acc_phase = 0, xph = 0;
        if (leader && unit < num_tiles) load_kv(unit);
        for (int t = unit; t < num_tiles; t += units, ++it) {
            const int m0 = row0(t), n0 = (t / num_m) * BN;
            // this CTA's rows of the tile that belong to its batch entry
            const int valid = max(0, min(BM, epi.x_rpb - (((t % num_m) % epi.x_mtpb) * TM + (int)rank * BM)));
            const bool live = row < valid && m0 + row < M;
            float rs = 1.0f;   // the fused RMSNorm of the query projection's input rows
            if (epi.rs_part && live) {
                float sum = 0.f;
                for (int tt = 0; tt < epi.rs_tiles; ++tt) sum += epi.rs_part[(int64_t)tt * epi.rs_ld + m0 + row];
                rs = rsqrtf(sum * epi.rs_inv_d + epi.rs_eps);
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (q == 2 && lane == 0) RF_TRACE(it, 4);
            // Q row -> bf16, K-major SW128 (two [128 rows][64 dims] halves)
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem + lane_base + (uint32_t)(acc * BN + c * 32), r);
                tmem_ld_wait();
                uint8_t *half = sQ + (c >> 1) * 16384 + row * 128;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const uint4 w = make_uint4(
                        pack_bf16(__uint_as_float(r[8 * qq]) * rs, __uint_as_float(r[8 * qq + 1]) * rs),
                        pack_bf16(__uint_as_float(r[8 * qq + 2]) * rs, __uint_as_float(r[8 * qq + 3]) * rs),
                        pack_bf16(__uint_as_float(r[8 * qq + 4]) * rs, __uint_as_float(r[8 * qq + 5]) * rs),
                        pack_bf16(__uint_as_float(r[8 * qq + 6]) * rs, __uint_as_float(r[8 * qq + 7]) * rs));
                    const int chunk = ((c & 1) * 4 + qq) ^ (row & 7);
                    *(uint4 *)(half + chunk * 16) = w;
                }
            }
            tc_fence_before();
            fence_proxy_async_smem();   // Q (generic proxy) -> visible to the tensor core
            __syncwarp();
            if (lane == 0) arrive_leader(&tempty[acc]);   // the accumulator is free for tile i + 2
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
            epi_sync();
            if (leader) arrive_leader(xq);
            if (issuer) {
                mbar_wait(xq, xph);
                mbar_wait(xk, xph);
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t ad = sdesc_sw128(sQ + (ks >> 2) * 16384) + (uint64_t)((ks & 3) * 2);
                    const uint64_t bd = sdesc_sw128(sK + (ks >> 2) * KV_HALF) + (uint64_t)((ks & 3) * 2);
                    if constexpr (CG == 2)
                        umma_bf16_pair(tmem + 256, ad, bd, idS, ks > 0);
                    else
                        umma_bf16(tmem + 256, ad, bd, idS, ks > 0);
                }
                if constexpr (CG == 2)
                    umma_commit_pair(xs);
                else
                    umma_commit(xs);
            }
            mbar_wait(xs, xph);
            tc_fence_after();
            uint32_t sr[128];
            tmem_ld32(tmem + lane_base + 256, *(uint32_t(*)[32])(sr));
            tmem_ld32(tmem + lane_base + 288, *(uint32_t(*)[32])(sr + 32));
            tmem_ld32(tmem + lane_base + 320, *(uint32_t(*)[32])(sr + 64));
            tmem_ld32(tmem + lane_base + 352, *(uint32_t(*)[32])(sr + 96));
            tmem_ld_wait();
            if (epi.x_nk < 128) {
#pragma unroll
                for (int e = 0; e < 128; ++e)
                    if (e >= epi.x_nk) sr[e] = __float_as_uint(-INFINITY);
            }
            float mx[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) mx[u] = fmaxf(__uint_as_float(sr[u]), __uint_as_float(sr[u + 4]));
#pragma unroll
            for (int e = 8; e < 128; e += 8)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    mx[u] = fmaxf(mx[u], fmaxf(__uint_as_float(sr[e + u]), __uint_as_float(sr[e + u + 4])));
            const float nm = -fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * epi.x_scale;
            float l = 0.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    float p0, p1;
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(fmaf(__uint_as_float(sr[c * 32 + 2 * e]), epi.x_scale, nm)));
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(fmaf(__uint_as_float(sr[c * 32 + 2 * e + 1]), epi.x_scale, nm)));
                    l += p0 + p1;
                    pk[e] = pack_bf16(p0, p1);
                }
                tmem_st16(tmem + lane_base + 256 + c * 16, pk);
            }
            tmem_st_wait();
            tc_fence_before();
            epi_sync();
            if (leader) arrive_leader(xp);
            if (issuer) {
                mbar_wait(xp, xph);
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t bd = sdesc_sw128(sV + (ks >> 2) * KV_HALF) + (uint64_t)((ks & 3) * 2);
                    if constexpr (CG == 2)
                        umma_bf16_ts_pair(tmem + 384, tmem + 256 + ks * 8, bd, idS, ks > 0);
                    else
                        umma_bf16_ts(tmem + 384, tmem + 256 + ks * 8, bd, idS, ks > 0);
                }
                if constexpr (CG == 2)
                    umma_commit_pair(xo);
                else
                    umma_commit(xo);
            }
            mbar_wait(xo, xph);
            tc_fence_after();
            xph ^= 1;
            // S and PV have read Q, K and V: prefetch the next tile's K / V^T
            if (leader && t + units < num_tiles) load_kv(t + units);
            const float inv_l = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem + lane_base + 384 + c * 32, r);
                tmem_ld_wait();
                uint4 pk[4];
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    pk[v] = make_uint4(
                        pack_bf16(__uint_as_float(r[v * 8]) * inv_l, __uint_as_float(r[v * 8 + 1]) * inv_l),
                        pack_bf16(__uint_as_float(r[v * 8 + 2]) * inv_l, __uint_as_float(r[v * 8 + 3]) * inv_l),
                        pack_bf16(__uint_as_float(r[v * 8 + 4]) * inv_l, __uint_as_float(r[v * 8 + 5]) * inv_l),
                        pack_bf16(__uint_as_float(r[v * 8 + 6]) * inv_l, __uint_as_float(r[v * 8 + 7]) * inv_l));
                // the tile's live rows: its batch entry's rows (valid), clipped at M
                store_rows_bf16x32((__nv_bfloat16 *)epi.out, epi.ldo, m0 + q * 32, m0 + min(valid, M - m0),
                                   n0 + c * 32, lane, pk);
            }
            tc_fence_before();
            epi_sync();   // O read by every warp before the next tile's PV overwrites it
            if (q == 2 && lane == 0) RF_TRACE(it, 5);
        }
    } else {
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int acc = 0, it = 0, t, kb0, kb1;
        uint32_t acc_phase = 0;
        for (Walk w = walk_init(); walk_next(w, t, kb0, kb1); ++it) {
            const int n0 = (t / num_m) * BN;
            {
            const int m0 = row0(t);
            const int m = m0 + q * 32 + lane;
            const bool live = m < M;
            float rs = 1.0f;   // fused RMSNorm of the A rows (kStoreBF16 with rs_part)
            if constexpr (EPI == kStoreBF16) {
                if (epi.rs_part && live) {
                    float sum = 0.f;
                    for (int t = 0; t < epi.rs_tiles; ++t) sum += epi.rs_part[(int64_t)t * epi.rs_ld + m];
                    rs = rsqrtf(sum * epi.rs_inv_d + epi.rs_eps);
                }
            }
            // kBF16Rope: this thread's token row of the (cos, sin) table, one 16-pair block
            // (8 float4) per 32-column chunk.  Chunks h * 128 + pb * 32 of the tile's heads
            // share block pb, so chunks are walked pb-major and block pb + 1 is prefetched
            // while block pb is applied (the table row is an L2 read; a load per use
            // stalled the epilogue behind the main loop).  Blocks 0 and 1 are loaded before
            // the accumulator wait, so their latency hides behind the tile's main loop (the
            // Q / K tiles' epilogue was longer than their main loop: tools/forward_timeline.py).
            constexpr int NCH = BN / 32;
            constexpr int NH = EPI == kBF16Rope ? BN / 128 : 1;
            if constexpr (C::TMA_O) {   // the previous tile's stores have read the staging buffer
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
            }
            float4 tc[8], tn[8];
            const float4 *tab = nullptr;
            bool tile_rot = false;
            if constexpr (EPI == kBF16Rope) {
                tile_rot = n0 < epi.rope_cols;
                tab = (const float4 *)(epi.rope + (int64_t)(m % epi.rows_per_batch) * 64);
                if (tile_rot) {
#pragma unroll
                    for (int v = 0; v < 8; ++v) tc[v] = __ldg(tab + v);
                    if (NH < NCH) {
#pragma unroll
                        for (int v = 0; v < 8; ++v) tn[v] = __ldg(tab + 8 + v);
                    }
                }
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (q == 2 && lane == 0) RF_TRACE(it, 4);
#pragma unroll 1
            for (int ci = 0; ci < NCH; ++ci) {
                const int c0 = EPI == kBF16Rope ? (ci % NH) * 128 + (ci / NH) * 32 : ci * 32;
                if constexpr (EPI == kBF16Rope) {
                    if (tile_rot && ci % NH == 0 && ci > 0) {   // block ci / NH is in tn
#pragma unroll
                        for (int v = 0; v < 8; ++v) tc[v] = tn[v];
                        if (ci + NH < NCH) {
#pragma unroll
                            for (int v = 0; v < 8; ++v) tn[v] = __ldg(tab + (ci / NH + 1) * 8 + v);
                        }
                    }
                }
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), r);
                tmem_ld_wait();
                // bf16 row stores are warp-collective (quad transposes): dead rows ride along
                if (!live && EPI != kStoreBF16 && EPI != kBF16Rope) continue;
                const int n = n0 + c0;
                if constexpr (EPI == kStoreBF16) {
                    uint4 pk[4];
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        uint32_t *p = (uint32_t *)&pk[v];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[v * 8 + 2 * e]) * rs,
                                                                     __uint_as_float(r[v * 8 + 2 * e + 1]) * rs);
                            p[e] = *(uint32_t *)&h;
                        }
                    }
                    store_rows_bf16x32((__nv_bfloat16 *)epi.out, epi.ldo, m0 + q * 32, M, n, lane, pk);
                } else if constexpr (EPI == kBF16Rope) {
                    const int nl = epi.vt_period ? n % epi.vt_period : n;
                    if (epi.vt && nl >= epi.vt_col0) {
                        const int cv = nl - epi.vt_col0, hv = cv >> 7, dim0 = cv & 127;
                        const int64_t b = m / epi.rows_per_batch, pos = m % epi.rows_per_batch;
                        const int64_t grp = epi.vt_period ? n / epi.vt_period : 0;
                        __nv_bfloat16 *dst = epi.vt + grp * epi.vt_layer_stride +
                                             ((b * epi.vt_heads + hv) * 128 + dim0) * epi.vt_ld + pos;
                        if (live) {
#pragma unroll
                            for (int e = 0; e < 32; ++e)   // lanes hold consecutive tokens: coalesced
                                dst[(int64_t)e * epi.vt_ld] = __float2bfloat16(__uint_as_float(r[e]));
                        }
                        continue;
                    }
                    const bool rot = n < epi.rope_cols;
                    uint4 pk4[4];
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        uint32_t *p = (uint32_t *)&pk4[v];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float x0 = __uint_as_float(r[v * 8 + 2 * e]), x1 = __uint_as_float(r[v * 8 + 2 * e + 1]);
                            if (rot) {
                                // q/k are bf16 Linear outputs: round, then rotate in fp32
                                x0 = bf16_round(x0);
                                x1 = bf16_round(x1);
                                const float4 c4 = tc[v * 2 + (e >> 1)];
                                const float2 c = (e & 1) ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
                                const float y0 = x0 * c.x - x1 * c.y, y1 = x0 * c.y + x1 * c.x;
                                x0 = y0;
                                x1 = y1;
                            }
                            __nv_bfloat162 hh = __floats2bfloat162_rn(x0, x1);
                            p[e] = *(uint32_t *)&hh;
                        }
                    }
                    store_rows_bf16x32((__nv_bfloat16 *)epi.out, epi.ldo, m0 + q * 32, M, n, lane, pk4);
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
                            y[h] = __fdividef(gt, 1.0f + __expf(-gt)) * up;   // fast divide: 2 ulp, far below bf16
                        }
                        __nv_bfloat162 hh = __floats2bfloat162_rn(y[0], y[1]);
                        p[e] = *(uint32_t *)&hh;
                    }
                    if constexpr (C::TMA_O) {
                        // output columns ci * 16 .. + 15: box ci / 4, 16-byte chunks 2 (ci % 4) + {0, 1}
                        uint8_t *box = sC + q * C::C_WARP_BYTES + (ci >> 2) * 4096 + lane * 128;
                        const int ch = (ci & 3) * 2;
                        *(uint4 *)(box + (((ch) ^ (lane & 7)) << 4)) = pk[0];
                        *(uint4 *)(box + (((ch + 1) ^ (lane & 7)) << 4)) = pk[1];
                    } else {
                        __nv_bfloat16 *o = (__nv_bfloat16 *)epi.out + (int64_t)m * epi.ldo + n / 2;
                        *(uint4 *)o = pk[0];
                        *(uint4 *)(o + 8) = pk[1];
                    }
                }
            }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2)
                    mbar_arrive_cluster(mapa_shared(&tempty[acc], 0));
                else
                    mbar_arrive(&tempty[acc]);
            }
            if (C::TMA_O) {   // rows >= M are clipped by the tensor map
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const int orow = row0(t) + q * 32;
                    tma_store_2d(&tma_c, sC + q * C::C_WARP_BYTES, n0 / 2, orow);
                    tma_store_2d(&tma_c, sC + q * C::C_WARP_BYTES + 4096, n0 / 2 + 64, orow);
                    bulk_commit();
                }
            }
            if (q == 2 && lane == 0) RF_TRACE(it, 5);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    if constexpr (C::TMA_O) {
        if (warp >= 2 && lane == 0) bulk_wait0();
    }
    if constexpr (CG == 2) {
        tc_fence_before();
        cluster_sync();   // the leader's MMAs and commits into this CTA are done
        if (warp == 1) tmem_dealloc_pair<TMEM_COLS>(tmem);
    } else {
        __syncthreads();
        if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
    }
    RF_GTRACE(14);
}

}  // namespace rf::gemm
