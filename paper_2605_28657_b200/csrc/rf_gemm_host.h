// Host-side GEMM plan (tensor maps built once, reused every launch).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rf {

struct GemmPlan {
    CUtensorMap ta, tb;
    int64_t M, N, K;
    int bn;
};

int make_tmap_bf16_2d(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                      uint32_t box_inner, uint32_t box_outer);
int gemm_plan(GemmPlan *p, const void *A, const void *B, int64_t M, int64_t N, int64_t K, int64_t lda,
              int64_t ldb, int bn);
// Transposed V output of the QKV / cross-KV GEMM (see EpiArgs::vt).
struct VtOut {
    void *ptr;
    int col0, heads;
    int64_t ld;
};

int gemm_run(const GemmPlan &p, int epi, void *out, int64_t ldo, const float *gate, int64_t gate_ld,
             int rows_per_batch, float alpha, cudaStream_t st, const float2 *rope = nullptr,
             int rope_cols = 0, int64_t M = 0, const VtOut *vt = nullptr);

// tcgen05 attention (rf_attention_tc.cu): tensor maps over Q, K and V^T built once.
struct AttnPlan {
    CUtensorMap tq, tk, tvt;
    int B, Nq, Nk, Nk_pad, H, Hkv;
};
int attn_plan(AttnPlan *p, const void *q, int64_t ldq_elems, int64_t q_cols, const void *k, int64_t ldk_elems,
              int64_t k_cols, const void *vt, int B, int Nq, int Nk, int Nk_pad, int H, int Hkv);
int attn_run(const AttnPlan &p, void *out, int64_t ldo, int B, cudaStream_t st);

}  // namespace rf
