// Host-side GEMM plan (tensor maps built once, reused every launch).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rf {

struct GemmPlan {
    CUtensorMap ta, tb;
    CUtensorMap tc;             // fp32 output map of the TMA-staged residual epilogue
    CUtensorMap tk, tvt;        // K / V^T maps of the cross-attention epilogue (RF_EPI_XATTN)
    void *c_ptr = nullptr;
    int64_t c_ld = 0, c_rows = 0;
    int64_t M, N, K;
    int bn;
    int cg;   // 1: 128 x bn tiles per CTA; 2: 256 x bn tiles per CTA pair (cta_group::2)
    bool b_static = false;   // B holds weights no kernel writes (see gemm::EpiArgs::b_static)
};

int make_tmap_bf16_2d(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                      uint32_t box_inner, uint32_t box_outer);
int make_tmap_f32_2d(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                     uint32_t box_inner, uint32_t box_outer);
// bind the residual-stream output of a kResidGate plan (builds its TMA map once)
int gemm_plan_c(GemmPlan *p, void *out, int64_t ldo);
// bind the bf16 output of a SwiGLU plan with 256-wide tiles (TMA-stored epilogue)
int gemm_plan_o(GemmPlan *p, void *out, int64_t ldo);
int gemm_plan(GemmPlan *p, const void *A, const void *B, int64_t M, int64_t N, int64_t K, int64_t lda,
              int64_t ldb, int bn, int cg = 1);
// Transposed V output of the QKV / cross-KV GEMM (see EpiArgs::vt).
struct VtOut {
    void *ptr;
    int col0, heads;
    int64_t ld;
    int period = 0;             // > 0: column groups of this width, one V^T block per group
    int64_t layer_stride = 0;   // elements between the groups' V^T blocks
};

// RMSNorm fused across a GEMM boundary (see gemm::EpiArgs): producer side (aux, sq_part) on
// a TMA-staged gated-residual GEMM, consumer side (rs_part) on a bf16-store GEMM.
struct NormFuse {
    void *aux = nullptr;
    int64_t aux_ld = 0;
    float *sq_part = nullptr;
    int64_t sq_ld = 0;
    const float *rs_part = nullptr;
    int64_t rs_ld = 0;
    int rs_tiles = 0;
    float rs_inv_d = 0.f, rs_eps = 0.f;
};

// Cross-attention in the query projection's epilogue (gemm::kCrossAttn): rows_per_batch
// query rows per batch entry, n_keys keys per entry, K / V^T through the attention maps.
struct XAttn {
    const CUtensorMap *tk, *tvt;
    const CUtensorMap *tk64, *tvt64;   // 64 x 64 boxes: one CTA's half of K / V^T on a CTA pair
    int rows_per_batch, batches, n_keys, group, kv_heads;
};

int gemm_run(const GemmPlan &p, int epi, void *out, int64_t ldo, const float *gate, int64_t gate_ld,
             int rows_per_batch, float alpha, cudaStream_t st, const float2 *rope = nullptr,
             int rope_cols = 0, int64_t M = 0, const VtOut *vt = nullptr, const NormFuse *nf = nullptr,
             const XAttn *xa = nullptr);

// tcgen05 attention (rf_attention_tc.cu): tensor maps over Q, K and V^T built once.
struct AttnPlan {
    CUtensorMap tq, tk, tvt, tk64;   // tk64: 64-key boxes (rf_attn_fa64_kernel)
    CUtensorMap tvt64;               // 64-key x 64-dim boxes (pair cross-attention epilogue)
    int B, Nq, Nk, Nk_pad, H, Hkv;
};
int attn_plan(AttnPlan *p, const void *q, int64_t ldq_elems, int64_t q_cols, const void *k, int64_t ldk_elems,
              int64_t k_cols, const void *vt, int B, int Nq, int Nk, int Nk_pad, int H, int Hkv);
int attn_run(const AttnPlan &p, void *out, int64_t ldo, int B, cudaStream_t st);

}  // namespace rf
