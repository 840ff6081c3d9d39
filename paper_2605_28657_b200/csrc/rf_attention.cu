// Multi-head attention forward (flash-attention-2 schedule) for the DiT: self-attention
// with grouped KV heads over a row's tokens, and cross-attention to conditioning tokens.
//
// One CTA = 4 warps = 64 query rows of one (batch row, head); K/V tiles of 64 keys are
// staged in XOR-swizzled shared memory by cp.async (double-buffered), S = Q K^T and
// O += P V run on bf16 tensor-core MMAs (m16n8k16, fp32 accumulate) with the online
// softmax kept in registers (exp2, scale folded).  Head dim 128.
//   q: [B*Nq, ldq] bf16, head h at column h*128;  k, v: [B*Nk, ldk] bf16, head h/group
//   out: [B*Nq, ldo] bf16, head h at column h*128.
#include "rf_common.cuh"

#include <cuda_bf16.h>

namespace rf {

constexpr int kAttnD = 128;
constexpr int kAttnBM = 64, kAttnBN = 64;
constexpr int kAttnThreads = 128;

struct AttnArgs {
    const __nv_bfloat16 *q, *k, *v;
    __nv_bfloat16 *out;
    int64_t ldq, ldk, ldv, ldo;
    int Nq, Nk, H, group;  // group = H / Hkv
    float scale_log2;      // log2(e) / sqrt(d)
};

__device__ __forceinline__ uint32_t swz(int row, int chunk) {  // byte offset in a 64 x 256 B tile
    return (uint32_t)(row * 256 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool pred) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                          uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *(uint32_t *)&h;
}

// stage rows [r0, r0+64) of a [N, ld] bf16 matrix (head columns col0..col0+127) into a tile
__device__ __forceinline__ void load_tile(uint32_t tile, const __nv_bfloat16 *base, int64_t ld, int r0, int N,
                                          int col0) {
    for (int i = threadIdx.x; i < 64 * 16; i += kAttnThreads) {
        const int row = i >> 4, chunk = i & 15;
        const int g = r0 + row;
        const bool ok = g < N;
        const __nv_bfloat16 *src = base + (int64_t)(ok ? g : 0) * ld + col0 + chunk * 8;
        cp_async16(tile + swz(row, chunk), src, ok);
    }
}

__global__ void __launch_bounds__(kAttnThreads)
rf_attention_kernel(const __grid_constant__ AttnArgs A) {
    extern __shared__ __align__(128) uint8_t sm[];
    const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t sK0 = sQ + 64 * 256, sV0 = sK0 + 2 * 64 * 256;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bh = blockIdx.y, b = bh / A.H, h = bh % A.H, hk = h / A.group;
    const int q0 = blockIdx.x * kAttnBM;
    const __nv_bfloat16 *qb = A.q + (int64_t)b * A.Nq * A.ldq;
    const __nv_bfloat16 *kb = A.k + (int64_t)b * A.Nk * A.ldk;
    const __nv_bfloat16 *vb = A.v + (int64_t)b * A.Nk * A.ldv;

    load_tile(sQ, qb, A.ldq, q0, A.Nq, h * kAttnD);
    cp_commit();
    const int ntiles = (A.Nk + kAttnBN - 1) / kAttnBN;
    load_tile(sK0, kb, A.ldk, 0, A.Nk, hk * kAttnD);
    load_tile(sV0, vb, A.ldv, 0, A.Nk, hk * kAttnD);
    cp_commit();

    // Q fragments: this warp's 16 rows x 128 dims (8 k-steps)
    cp_wait<1>();
    __syncthreads();
    uint32_t qf[8][4];
    {
        const int row = warp * 16 + (lane & 15);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int chunk = ks * 2 + (lane >> 4);
            ldsm_x4(sQ + swz(row, chunk), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
        }
    }
    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};

    for (int t = 0; t < ntiles; ++t) {
        const int buf = t & 1;
        if (t + 1 < ntiles) {
            load_tile(sK0 + (buf ^ 1) * 64 * 256, kb, A.ldk, (t + 1) * kAttnBN, A.Nk, hk * kAttnD);
            load_tile(sV0 + (buf ^ 1) * 64 * 256, vb, A.ldv, (t + 1) * kAttnBN, A.Nk, hk * kAttnD);
        }
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const uint32_t sK = sK0 + buf * 64 * 256, sV = sV0 + buf * 64 * 256;
        // S = Q K^T : 16 x 64 per warp (8 n-tiles of 8 keys)
        float s[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) {  // pairs of n-tiles (16 keys)
                const int key = jp * 16 + (lane & 7) + ((lane >> 4) << 3);
                const int chunk = ks * 2 + ((lane >> 3) & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sK + swz(key, chunk), b0, b1, b2, b3);
                mma16816(s[2 * jp], qf[ks], b0, b1);
                mma16816(s[2 * jp + 1], qf[ks], b2, b3);
            }
        }
        // mask keys beyond Nk, online softmax (rows g and g+8 of this warp)
        const int kbase = t * kAttnBN;
        float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = kbase + j * 8 + 2 * (lane & 3) + (e & 1);
                float v = s[j][e] * A.scale_log2;
                if (key >= A.Nk) v = -INFINITY;
                s[j][e] = v;
                mnew[e >> 1] = fmaxf(mnew[e >> 1], v);
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 1));
            mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 2));
        }
        float corr[2], rsum[2] = {0.f, 0.f};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            corr[r] = mrow[r] == -INFINITY ? 0.f : exp2f(mrow[r] - mnew[r]);
            mrow[r] = mnew[r];
        }
        uint32_t pf[4][4];  // P as A fragments, 4 k-steps of 16 keys
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                p[e] = mrow[e >> 1] == -INFINITY ? 0.f : exp2f(s[j][e] - mrow[e >> 1]);
                rsum[e >> 1] += p[e];
            }
            pf[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
            pf[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) lrow[r] = lrow[r] * corr[r] + rsum[r];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            o[i][0] *= corr[0];
            o[i][1] *= corr[0];
            o[i][2] *= corr[1];
            o[i][3] *= corr[1];
        }
        // O += P V : 16 x 128 per warp (16 dim tiles), 4 k-steps of 16 keys
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            uint32_t a[4] = {pf[ks][0], pf[ks][1], pf[ks][2], pf[ks][3]};
#pragma unroll
            for (int dp = 0; dp < 8; ++dp) {  // pairs of dim tiles (16 dims)
                const int key = ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
                const int chunk = dp * 2 + (lane >> 4);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(sV + swz(key, chunk), b0, b1, b2, b3);
                mma16816(o[2 * dp], a, b0, b1);
                mma16816(o[2 * dp + 1], a, b2, b3);
            }
        }
        __syncthreads();  // buffer `buf` is reloaded at iteration t + 1
    }
    // normalise and store
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        float l = lrow[r];
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        lrow[r] = l > 0.f ? 1.f / l : 0.f;
    }
    const int g = lane >> 2, tq = lane & 3;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int qrow = q0 + warp * 16 + g + r * 8;
        if (qrow >= A.Nq) continue;
        __nv_bfloat16 *dst = A.out + ((int64_t)b * A.Nq + qrow) * A.ldo + h * kAttnD;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const uint32_t pk = pack_bf16(o[i][2 * r] * lrow[r], o[i][2 * r + 1] * lrow[r]);
            *(uint32_t *)(dst + i * 8 + 2 * tq) = pk;
        }
    }
}

}  // namespace rf

using namespace rf;

extern "C" int rf_attention_bf16(const void *q, const void *k, const void *v, void *out, int32_t batch,
                                 int32_t n_q, int32_t n_k, int32_t heads, int32_t kv_heads, int64_t ldq,
                                 int64_t ldk, int64_t ldv, int64_t ldo, void *stream) {
    if (!q || !k || !v || !out || batch < 1 || n_q < 1 || n_k < 1 || heads < 1 || kv_heads < 1 ||
        heads % kv_heads) {
        set_error("rf_attention_bf16: bad arguments");
        return RF_EINVAL;
    }
    AttnArgs A{(const __nv_bfloat16 *)q, (const __nv_bfloat16 *)k, (const __nv_bfloat16 *)v,
               (__nv_bfloat16 *)out, ldq, ldk, ldv, ldo, n_q, n_k, heads, heads / kv_heads,
               1.4426950408889634f / sqrtf((float)kAttnD)};
    const int smem = 64 * 256 * 5;  // Q + 2 x (K, V)
    static bool attr = false;
    if (!attr) {
        RF_TRY_CUDA(cudaFuncSetAttribute(rf_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    dim3 grid((n_q + kAttnBM - 1) / kAttnBM, batch * heads);
    rf_attention_kernel<<<grid, kAttnThreads, smem, (cudaStream_t)stream>>>(A);
    RF_TRY_LAUNCH("rf_attention_kernel");
    return RF_OK;
}
