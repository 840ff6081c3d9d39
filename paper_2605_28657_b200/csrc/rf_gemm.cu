// Host side of the tcgen05 GEMM: TMA tensor maps and launches (see rf_gemm.cuh).
#include "rf_common.cuh"
#include "rf_gemm.cuh"
#include "rf_gemm_host.h"

namespace rf {

typedef CUresult (*PFN_tmapEncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                        const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                        const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_tmapEncodeTiled encode_fn() {
    static PFN_tmapEncodeTiled fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_tmapEncodeTiled)p;
    }
    return fn;
}

static int make_tmap_2d(CUtensorMap *map, CUtensorMapDataType dt, const void *ptr, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer);

int make_tmap_bf16_2d(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                      uint32_t box_inner, uint32_t box_outer) {
    return make_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, ptr, inner, outer, row_bytes, box_inner, box_outer);
}

int make_tmap_f32_2d(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                     uint32_t box_inner, uint32_t box_outer) {
    return make_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, ptr, inner, outer, row_bytes, box_inner, box_outer);
}

static int make_tmap_2d(CUtensorMap *map, CUtensorMapDataType dt, const void *ptr, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
    PFN_tmapEncodeTiled enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return RF_ECUDA;
    }
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    // TMA fetches promoted to 256-byte L2 lines (measured +0.3-0.4% over 128 B / none)
    const CUtensorMapL2promotion pr = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    CUresult r = enc(map, dt, 2, const_cast<void *>(ptr), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu stride=%llu", (int)r,
                  (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_bytes);
        return RF_ECUDA;
    }
    return RF_OK;
}

template <int BN, int EPI, int CG, int CC = BN>
static int launch(const GemmPlan &p, const gemm::EpiArgs &e, cudaStream_t st) {
    using C = gemm::Cfg<BN, CG, EPI, CC>;
    auto kern = gemm::rf_gemm_kernel<BN, EPI, CG, CC>;
    static bool attr = false;
    if (!attr) {
        RF_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
        attr = true;
    }
    const int tiles = (EPI == gemm::kCrossAttn ? e.x_batches * e.x_mtpb
                                               : (int)((p.M + gemm::BM * CG - 1) / (gemm::BM * CG))) *
                      (int)(p.N / BN);
    int units = sm_count() / CG;   // persistent: one CTA (pair) per SM (pair)
    if (tiles < units) units = tiles;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(units * CG));
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[3];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see pdl_wait()
    at[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = CG;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = add_l2_window(at, CG == 2 ? 2 : 1);
    RF_TRY_CUDA(cudaLaunchKernelEx(&cfg, kern, p.ta, p.tb, p.tc, p.tk, p.tvt, (int)p.M, (int)p.N, (int)p.K, e));
    RF_TRY_LAUNCH("rf_gemm_kernel");
    return RF_OK;
}

template <int BN, int CG>
static int dispatch(const GemmPlan &p, int epi, const gemm::EpiArgs &e, cudaStream_t st) {
    switch (epi) {
        case gemm::kStoreBF16: return launch<BN, gemm::kStoreBF16, CG>(p, e, st);
        case gemm::kStoreF32: return launch<BN, gemm::kStoreF32, CG>(p, e, st);
        case gemm::kResidGate:
            // long K: the main loop hides a two-pass residual epilogue; keep the operand stages
            // (256-wide tiles always stage 64 columns per pass)
            if constexpr (BN == 256) {
                return launch<BN, gemm::kResidGate, CG, 64>(p, e, st);
            } else {
                // long K (the down projection, K = 6144): the residual staged 32 columns per
                // pass leaves room for an 8th operand stage, which the 96-k-block main loop's
                // feed needs more than the epilogue needs the staging (61.2 vs 62.9 us
                // standalone, profiles/r2_gemm_trace.txt); K = 2048 keeps one 128-column pass
                if (p.K >= 4096) return launch<BN, gemm::kResidGate, CG, 32>(p, e, st);
                return launch<BN, gemm::kResidGate, CG>(p, e, st);
            }
        case gemm::kSwiGLU: return launch<BN, gemm::kSwiGLU, CG>(p, e, st);
        case gemm::kStoreF32Scale: return launch<BN, gemm::kStoreF32Scale, CG>(p, e, st);
        case gemm::kBF16Rope: return launch<BN, gemm::kBF16Rope, CG>(p, e, st);
    }
    set_error("gemm: bad epilogue %d", epi);
    return RF_EINVAL;
}

int gemm_plan(GemmPlan *p, const void *A, const void *B, int64_t M, int64_t N, int64_t K, int64_t lda,
              int64_t ldb, int bn, int cg) {
    if (K % gemm::BK || (bn != 128 && bn != 256) || (cg != 1 && cg != 2) || N % bn || M < 1) {
        set_error("gemm: unsupported shape M=%lld N=%lld K=%lld BN=%d CG=%d", (long long)M, (long long)N,
                  (long long)K, bn, cg);
        return RF_EINVAL;
    }
    p->M = M;
    p->N = N;
    p->K = K;
    p->bn = bn;
    p->cg = cg;
    int rc = make_tmap_bf16_2d(&p->ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda * 2, gemm::BK, gemm::BM);
    if (rc) return rc;
    return make_tmap_bf16_2d(&p->tb, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb * 2, gemm::BK, (uint32_t)(bn / cg));
}

static unsigned long long *g_trace = nullptr;   // debugging timeline buffer (rf_gemm_set_trace)
// sequential mode (rf_gemm_set_trace_seq): launch i gets its own [cta][16][8] block
static int64_t g_trace_seq_max = 0, g_trace_seq_next = 0;
constexpr int64_t kTraceBlock = 400 * 16 * 8;

int gemm_plan_c(GemmPlan *p, void *out, int64_t ldo) {
    p->c_ptr = out;
    p->c_ld = ldo;
    p->c_rows = p->M;   // stores clip at M rows
    // fp32 [M, N] with row stride ldo, 32 x 32 boxes (128-byte rows: SWIZZLE_128B)
    return make_tmap_f32_2d(&p->tc, out, (uint64_t)p->N, (uint64_t)p->M, (uint64_t)ldo * 4, 32, 32);
}

int gemm_plan_o(GemmPlan *p, void *out, int64_t ldo) {
    p->c_ptr = out;
    p->c_ld = ldo;
    p->c_rows = p->M;
    // bf16 [M, N / 2] SwiGLU output, 64 x 32 boxes (128-byte rows: SWIZZLE_128B)
    return make_tmap_bf16_2d(&p->tc, out, (uint64_t)(p->N / 2), (uint64_t)p->M, (uint64_t)ldo * 2, 64, 32);
}

int gemm_run(const GemmPlan &plan, int epi, void *out, int64_t ldo, const float *gate, int64_t gate_ld,
             int rows_per_batch, float alpha, cudaStream_t st, const float2 *rope, int rope_cols, int64_t M,
             const VtOut *vt, const NormFuse *nf, const XAttn *xa) {
    // The tensor maps cover the plan's (maximum) M; a smaller M only shortens the tile walk.
    GemmPlan p = plan;
    if (M > 0 && M < p.M) p.M = M;
    if (epi == gemm::kResidGate && (p.c_ptr != out || p.c_ld != ldo || p.c_rows != p.M)) {
        // the TMA-staged residual epilogue needs a map over `out` (cached when planned)
        int rc = gemm_plan_c(&p, out, ldo);
        if (rc) return rc;
    }
    if (epi == gemm::kSwiGLU && p.bn == 256 && (p.c_ptr != out || p.c_ld != ldo || p.c_rows != p.M)) {
        // the TMA-stored SwiGLU epilogue needs a map over `out` (cached when planned)
        int rc = gemm_plan_o(&p, out, ldo);
        if (rc) return rc;
    }
    gemm::EpiArgs e{out, ldo, gate, gate_ld, rows_per_batch > 0 ? rows_per_batch : 1, alpha, rope, rope_cols,
                    vt ? (__nv_bfloat16 *)vt->ptr : nullptr, vt ? vt->col0 : 0, vt ? vt->heads : 0,
                    vt ? vt->ld : 0, vt ? vt->period : 0, vt ? vt->layer_stride : 0, g_trace};
    e.b_static = p.b_static ? 1 : 0;
    if (g_trace && g_trace_seq_max > 0)   // each launch (also each captured graph node) its own block
        e.trace = g_trace_seq_next < g_trace_seq_max ? g_trace + kTraceBlock * g_trace_seq_next++ : nullptr;
    if (nf) {
        if ((nf->aux && epi != gemm::kResidGate) || (nf->rs_part && epi != gemm::kStoreBF16 && epi != gemm::kCrossAttn)) {
            set_error("gemm: fused norm needs a gated-residual producer / bf16-store consumer");
            return RF_EINVAL;
        }
        e.aux = (__nv_bfloat16 *)nf->aux;
        e.aux_ld = nf->aux_ld;
        e.sq_part = nf->sq_part;
        e.sq_ld = nf->sq_ld;
        e.rs_part = nf->rs_part;
        e.rs_ld = nf->rs_ld;
        e.rs_tiles = nf->rs_tiles;
        e.rs_inv_d = nf->rs_inv_d;
        e.rs_eps = nf->rs_eps;
    }
    if (epi == gemm::kCrossAttn) {
        if (!xa || p.bn != 128 || xa->n_keys > 128 || xa->n_keys < 1 || xa->rows_per_batch < 1 || p.N % 128 ||
            (p.cg == 2 && (!xa->tk64 || !xa->tvt64))) {
            set_error("gemm: cross-attention epilogue needs 128-wide tiles and <= 128 keys");
            return RF_EINVAL;
        }
        p.tk = p.cg == 2 ? *xa->tk64 : *xa->tk;
        p.tvt = p.cg == 2 ? *xa->tvt64 : *xa->tvt;
        e.x_rpb = xa->rows_per_batch;
        e.x_mtpb = (xa->rows_per_batch + gemm::BM * p.cg - 1) / (gemm::BM * p.cg);
        e.x_batches = xa->batches;
        e.x_nk = xa->n_keys;
        e.x_group = xa->group;
        e.x_hkv = xa->kv_heads;
        e.x_scale = 1.4426950408889634f / sqrtf(128.f);
        if (p.cg == 2) return launch<128, gemm::kCrossAttn, 2>(p, e, st);
        return launch<128, gemm::kCrossAttn, 1>(p, e, st);
    }
    if (p.bn == 256) return p.cg == 2 ? dispatch<256, 2>(p, epi, e, st) : dispatch<256, 1>(p, epi, e, st);
    return p.cg == 2 ? dispatch<128, 2>(p, epi, e, st) : dispatch<128, 1>(p, epi, e, st);
}

}  // namespace rf

using namespace rf;

// Debugging aid (not part of the product ABI): when set, every GEMM launch records a
// clock64 timeline per CTA into buf ([cta][tile < 16][8] u64) -- see tools/gemm_trace.py.
extern "C" void rf_gemm_set_trace(void *buf) {
    g_trace = (unsigned long long *)buf;
    g_trace_seq_max = 0;
}
// Debugging aid: every GEMM launched (or captured into a graph) from now on records its
// per-CTA entry / exit globaltimer stamps in its own block of buf ([launch][400][16][8] u64,
// entry at [cta][15][7], exit at [cta][14][7]) -- the in-situ timeline of a DiT forward
// (tools/forward_timeline.py).  Returns the launch index the next GEMM will get.
extern "C" int64_t rf_gemm_set_trace_seq(void *buf, int64_t max_launches) {
    g_trace = (unsigned long long *)buf;
    g_trace_seq_max = buf ? max_launches : 0;
    g_trace_seq_next = 0;
    return 0;
}

extern "C" int rf_gemm_bf16(const void *A, const void *B, void *out, int64_t M, int64_t N, int64_t K,
                            int64_t lda, int64_t ldb, int64_t ldo, int32_t epilogue, const float *gate,
                            int64_t gate_ld, int32_t rows_per_batch, float alpha, int32_t block_n,
                            void *stream) {
    // block_n: 128 / 256 = one CTA per 128 x block_n tile; -128 / -256 = a CTA pair
    // (cta_group::2) per 256 x |block_n| tile
    if (!A || !B || !out || (epilogue == gemm::kResidGate && !gate) || epilogue == gemm::kBF16Rope) {
        set_error("rf_gemm_bf16: null argument");
        return RF_EINVAL;
    }
    GemmPlan p;
    const int mag = block_n < 0 ? -block_n : block_n;
    int rc = gemm_plan(&p, A, B, M, N, K, lda, ldb, mag, block_n < 0 ? 2 : 1);
    if (rc) return rc;
    return gemm_run(p, epilogue, out, ldo, gate, gate_ld, rows_per_batch, alpha, (cudaStream_t)stream);
}
