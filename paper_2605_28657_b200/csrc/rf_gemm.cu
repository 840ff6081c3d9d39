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

int make_tmap_bf16_2d(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                      uint32_t box_inner, uint32_t box_outer) {
    PFN_tmapEncodeTiled enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return RF_ECUDA;
    }
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu stride=%llu", (int)r,
                  (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_bytes);
        return RF_ECUDA;
    }
    return RF_OK;
}

template <int BN, int EPI>
static int launch(const GemmPlan &p, const gemm::EpiArgs &e, cudaStream_t st) {
    using C = gemm::Cfg<BN>;
    auto kern = gemm::rf_gemm_kernel<BN, EPI>;
    static bool attr = false;
    if (!attr) {
        RF_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
        attr = true;
    }
    const int tiles = (int)((p.M + gemm::BM - 1) / gemm::BM) * (int)(p.N / BN);
    int grid = sm_count();
    if (tiles < grid) grid = tiles;
    kern<<<grid, 192, C::SMEM, st>>>(p.ta, p.tb, (int)p.M, (int)p.N, (int)p.K, e);
    RF_TRY_LAUNCH("rf_gemm_kernel");
    return RF_OK;
}

int gemm_plan(GemmPlan *p, const void *A, const void *B, int64_t M, int64_t N, int64_t K, int64_t lda,
              int64_t ldb, int bn) {
    if (K % gemm::BK || (bn != 128 && bn != 256) || N % bn || M < 1) {
        set_error("gemm: unsupported shape M=%lld N=%lld K=%lld BN=%d", (long long)M, (long long)N,
                  (long long)K, bn);
        return RF_EINVAL;
    }
    p->M = M;
    p->N = N;
    p->K = K;
    p->bn = bn;
    int rc = make_tmap_bf16_2d(&p->ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda * 2, gemm::BK, gemm::BM);
    if (rc) return rc;
    return make_tmap_bf16_2d(&p->tb, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb * 2, gemm::BK, (uint32_t)bn);
}

int gemm_run(const GemmPlan &plan, int epi, void *out, int64_t ldo, const float *gate, int64_t gate_ld,
             int rows_per_batch, float alpha, cudaStream_t st, const float2 *rope, int rope_cols, int64_t M,
             const VtOut *vt) {
    // The tensor maps cover the plan's (maximum) M; a smaller M only shortens the tile walk.
    GemmPlan p = plan;
    if (M > 0 && M < p.M) p.M = M;
    gemm::EpiArgs e{out, ldo, gate, gate_ld, rows_per_batch > 0 ? rows_per_batch : 1, alpha, rope, rope_cols,
                    vt ? (__nv_bfloat16 *)vt->ptr : nullptr, vt ? vt->col0 : 0, vt ? vt->heads : 0,
                    vt ? vt->ld : 0};
    if (p.bn == 256) {
        switch (epi) {
            case gemm::kStoreBF16: return launch<256, gemm::kStoreBF16>(p, e, st);
            case gemm::kStoreF32: return launch<256, gemm::kStoreF32>(p, e, st);
            case gemm::kResidGate: return launch<256, gemm::kResidGate>(p, e, st);
            case gemm::kSwiGLU: return launch<256, gemm::kSwiGLU>(p, e, st);
            case gemm::kStoreF32Scale: return launch<256, gemm::kStoreF32Scale>(p, e, st);
            case gemm::kBF16Rope: return launch<256, gemm::kBF16Rope>(p, e, st);
        }
    } else {
        switch (epi) {
            case gemm::kStoreBF16: return launch<128, gemm::kStoreBF16>(p, e, st);
            case gemm::kStoreF32: return launch<128, gemm::kStoreF32>(p, e, st);
            case gemm::kResidGate: return launch<128, gemm::kResidGate>(p, e, st);
            case gemm::kSwiGLU: return launch<128, gemm::kSwiGLU>(p, e, st);
            case gemm::kStoreF32Scale: return launch<128, gemm::kStoreF32Scale>(p, e, st);
            case gemm::kBF16Rope: return launch<128, gemm::kBF16Rope>(p, e, st);
        }
    }
    set_error("gemm: bad epilogue %d", epi);
    return RF_EINVAL;
}

}  // namespace rf

using namespace rf;

extern "C" int rf_gemm_bf16(const void *A, const void *B, void *out, int64_t M, int64_t N, int64_t K,
                            int64_t lda, int64_t ldb, int64_t ldo, int32_t epilogue, const float *gate,
                            int64_t gate_ld, int32_t rows_per_batch, float alpha, int32_t block_n,
                            void *stream) {
    if (!A || !B || !out || (epilogue == gemm::kResidGate && !gate) || epilogue == gemm::kBF16Rope) {
        set_error("rf_gemm_bf16: null argument");
        return RF_EINVAL;
    }
    GemmPlan p;
    int rc = gemm_plan(&p, A, B, M, N, K, lda, ldb, block_n);
    if (rc) return rc;
    return gemm_run(p, epilogue, out, ldo, gate, gate_ld, rows_per_batch, alpha, (cudaStream_t)stream);
}
