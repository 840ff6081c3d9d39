// Admission init, emit statistics and deterministic squared-difference reductions
// (SURVEY.md §8(a) A16, A17).
#include <math.h>

#include "rf_common.cuh"

namespace rf {

constexpr int kRedThreads = 256;
constexpr int kRedPairs = 2;                             // double2 loads per thread
constexpr int kRedChunk = kRedThreads * 2 * kRedPairs;  // elements per block (1024)
constexpr int kMaxEmit = 16;
constexpr int kMaxAdmit = 32;

struct AdmitBatch {
    int count;
    rf_admit a[kMaxAdmit];
};

// _admit (pipeline.py:523-532): x = noise, or d*noise + (1-d)*source.
__global__ void rf_admit_kernel(const __grid_constant__ AdmitBatch B, int64_t numel) {
    pdl_wait();
    pdl_launch();
    const rf_admit &A = B.a[blockIdx.y];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel;
         i += (int64_t)gridDim.x * blockDim.x) {
        double n = A.noise[i];
        A.x[i] = A.source ? __dadd_rn(__dmul_rn(A.denoise, n), __dmul_rn(__dsub_rn(1.0, A.denoise), A.source[i]))
                          : n;
    }
}

// Fixed-shape reduction tree: each thread sums its kRedPairs coalesced double2 pairs in
// order, then a fixed shuffle/shared tree per block, then a fixed warp tree over the blocks'
// partials.  The result depends only on numel, never on timing.
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) {
        for (int w = 0; w < kRedThreads / 32; ++w) r = __dadd_rn(r, sh[w]);
    }
    __syncthreads();
    return r;
}

// one warp per emit: lane-strided sums of the block partials, then a fixed shuffle tree
__device__ __forceinline__ double warp_sum_fixed(const double *part, int64_t chunks) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int64_t c = lane; c < chunks; c += 32) s = __dadd_rn(s, __ldcg(part + c));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
    return s;
}

struct EmitBatch {
    int count;
    rf_emit e[kMaxEmit];
};

// grid (chunks, emits): copy latent -> record, isfinite flag, chunk partials of
// (lat - prev)^2 and (lat - ref)^2; the last block of each emit to finish (a counter per
// emit, left zero again) sums that emit's partials with the fixed warp tree and writes its
// mse values -- no second launch.
__global__ void __launch_bounds__(kRedThreads)
rf_emit_partials(const __grid_constant__ EmitBatch B, int64_t numel, const double *__restrict__ last,
                 const double *__restrict__ ref, double *__restrict__ part_prev,
                 double *__restrict__ part_ref, uint32_t *__restrict__ status, unsigned int *__restrict__ done,
                 double *__restrict__ mse_prev, double *__restrict__ mse_ref, int has_last) {
    __shared__ double sh[kRedThreads / 32];
    __shared__ bool last_block;
    pdl_wait();
    pdl_launch();
    const int e = blockIdx.y;
    const double *lat = B.e[e].latent;
    double *rec = B.e[e].record;
    const double *prev = e == 0 ? last : B.e[e - 1].latent;
    // pair k of thread t: elements base + 2 (k * kRedThreads + t) + {0, 1} (coalesced)
    const int64_t base = (int64_t)blockIdx.x * kRedChunk;
    double sp = 0.0, sr = 0.0;
    bool bad = false;
    double lv[kRedPairs][2], pv[kRedPairs][2], rv[kRedPairs][2];
#pragma unroll
    for (int k = 0; k < kRedPairs; ++k) {   // every load first: one memory round trip
        const int64_t i = base + 2 * ((int64_t)k * kRedThreads + threadIdx.x);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool in = i + h < numel;
            lv[k][h] = in ? lat[i + h] : 0.0;
            pv[k][h] = in && prev ? prev[i + h] : 0.0;
            rv[k][h] = in && ref ? ref[i + h] : 0.0;
        }
    }
#pragma unroll
    for (int k = 0; k < kRedPairs; ++k) {
        const int64_t i = base + 2 * ((int64_t)k * kRedThreads + threadIdx.x);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (i + h >= numel) continue;
            const double v = lv[k][h];
            rec[i + h] = v;
            if (!isfinite(v)) bad = true;
            if (prev) {
                double d = __dsub_rn(v, pv[k][h]);
                sp = __dadd_rn(sp, __dmul_rn(d, d));
            }
            if (ref) {
                double d = __dsub_rn(v, rv[k][h]);
                sr = __dadd_rn(sr, __dmul_rn(d, d));
            }
        }
    }
    if (bad) atomicOr(status, RF_STATUS_NONFINITE);
    double bp = block_sum(sp, sh);
    double br = block_sum(sr, sh);
    if (threadIdx.x == 0) {
        part_prev[(int64_t)e * gridDim.x + blockIdx.x] = bp;
        part_ref[(int64_t)e * gridDim.x + blockIdx.x] = br;
        __threadfence();
        last_block = atomicAdd(done + e, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last_block || threadIdx.x >= 32) return;
    __threadfence();
    const int64_t chunks = gridDim.x;
    const double tp = warp_sum_fixed(part_prev + e * chunks, chunks);
    const double tr = warp_sum_fixed(part_ref + e * chunks, chunks);
    if (threadIdx.x == 0) {
        // prev of emit 0 is `last` (may be absent); later emits always have a prev
        mse_prev[e] = (e == 0 && !has_last) ? -1.0 : __ddiv_rn(tp, (double)numel);
        mse_ref[e] = ref ? __ddiv_rn(tr, (double)numel) : -1.0;
        done[e] = 0u;   // ready for the next launch
    }
}

}  // namespace rf

using namespace rf;

extern "C" int rf_admit_init(const rf_admit *admits, int count, int64_t numel, void *stream) {
    if (count <= 0) return RF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    for (int c0 = 0; c0 < count; c0 += kMaxAdmit) {
        AdmitBatch B;
        B.count = count - c0 < kMaxAdmit ? count - c0 : kMaxAdmit;
        for (int i = 0; i < B.count; ++i) {
            B.a[i] = admits[c0 + i];
            if (!B.a[i].x || !B.a[i].noise) {
                set_error("rf_admit_init: null pointer in admit %d", c0 + i);
                return RF_EINVAL;
            }
        }
        int64_t bx = (numel + 255) / 256;
        if (bx > 1024) bx = 1024;
        RF_TRY_CUDA(launch_pdl(rf_admit_kernel, dim3((unsigned)bx, (unsigned)B.count), dim3(256), 0, st, B, numel));
        RF_TRY_LAUNCH("rf_admit_kernel");
    }
    return RF_OK;
}

__global__ void rf_x0_kernel(double *out, const double *base, const double *hint, double hs,
                             const double *timbre, double ts, const double *style, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v = base[i];
        if (hint) v = __dadd_rn(v, __dmul_rn(hs, hint[i]));
        if (timbre) v = __dadd_rn(v, __dmul_rn(ts, timbre[i]));
        if (style) v = __dadd_rn(v, style[i]);
        out[i] = v;
    }
}

extern "C" int rf_x0_compose(double *out, const double *base, const double *hint, double hs,
                             const double *timbre, double ts, const double *style, int64_t numel,
                             void *stream) {
    if (!out || !base || numel <= 0) {
        set_error("rf_x0_compose: bad arguments");
        return RF_EINVAL;
    }
    int64_t bx = (numel + 255) / 256;
    if (bx > 4096) bx = 4096;
    rf_x0_kernel<<<(unsigned)bx, 256, 0, (cudaStream_t)stream>>>(out, base, hint, hs, timbre, ts, style,
                                                                  numel);
    RF_TRY_LAUNCH("rf_x0_kernel");
    return RF_OK;
}

// Reduction scratch is the caller's (one buffer per stream: concurrent pipelines and
// devices never share partials).  Emits are processed in chunks of kMaxEmit launches;
// chunk c's first "previous latent" is chunk c-1's last latent, so any number of
// completions per tick (any ring depth) gives the same statistics as one batch.
extern "C" int64_t rf_reduce_workspace_elems(int64_t numel) {
    if (numel <= 0) return 0;
    const int64_t chunks = (numel + kRedChunk - 1) / kRedChunk;
    return 2 * chunks * kMaxEmit + kMaxEmit;   // partials, then kMaxEmit completion counters
}

extern "C" int rf_emit_stats(const rf_emit *emits, int count, int64_t numel, const double *last,
                             const double *reference, double *mse_prev, double *mse_ref,
                             uint32_t *status, double *scratch, int64_t scratch_elems, void *stream) {
    if (count <= 0) return RF_OK;
    if (!emits || !mse_prev || !mse_ref || !status || numel <= 0 || !scratch) {
        set_error("rf_emit_stats: bad arguments (count %d)", count);
        return RF_EINVAL;
    }
    if (scratch_elems < rf_reduce_workspace_elems(numel)) {
        set_error("rf_emit_stats: scratch of %lld doubles < %lld", (long long)scratch_elems,
                  (long long)rf_reduce_workspace_elems(numel));
        return RF_EWORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t chunks = (numel + kRedChunk - 1) / kRedChunk;
    double *pp = scratch, *pr = scratch + chunks * kMaxEmit;
    // the per-emit completion counters (zero before the first call; every launch leaves them zero)
    unsigned int *done = (unsigned int *)(scratch + 2 * chunks * kMaxEmit);
    for (int c0 = 0; c0 < count; c0 += kMaxEmit) {
        EmitBatch B;
        B.count = count - c0 < kMaxEmit ? count - c0 : kMaxEmit;
        for (int i = 0; i < B.count; ++i) {
            B.e[i] = emits[c0 + i];
            if (!B.e[i].latent || !B.e[i].record) {
                set_error("rf_emit_stats: null pointer in emit %d", c0 + i);
                return RF_EINVAL;
            }
        }
        const double *prev = c0 == 0 ? last : emits[c0 - 1].latent;
        RF_TRY_CUDA(launch_pdl(rf_emit_partials, dim3((unsigned)chunks, (unsigned)B.count), dim3(kRedThreads), 0, st,
                               B, numel, prev, reference, pp, pr, status, done, mse_prev + c0, mse_ref + c0,
                               (int)(prev != nullptr)));
        RF_TRY_LAUNCH("rf_emit_partials");
    }
    return RF_OK;
}

// mse of two arrays with the same fixed-order tree (used by the Python seams).
__global__ void __launch_bounds__(kRedThreads)
rf_sqdiff_partials(const double *__restrict__ a, const double *__restrict__ b, int64_t numel,
                   double *__restrict__ part) {
    __shared__ double sh[kRedThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kRedChunk;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kRedPairs; ++k) {
        const int64_t i = base + 2 * ((int64_t)k * kRedThreads + threadIdx.x);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (i + h < numel) {
                double d = __dsub_rn(a[i + h], b[i + h]);
                s = __dadd_rn(s, __dmul_rn(d, d));
            }
        }
    }
    double r = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = r;
}

__global__ void rf_sum_finish(const double *part, int64_t chunks, int64_t numel, double *out) {
    const double s = warp_sum_fixed(part, chunks);
    if (threadIdx.x == 0) *out = __ddiv_rn(s, (double)numel);
}

extern "C" int rf_mse(const double *a, const double *b, int64_t numel, double *out, double *scratch,
                      int64_t scratch_elems, void *stream) {
    if (!a || !b || !out || numel <= 0 || !scratch) {
        set_error("rf_mse: bad arguments");
        return RF_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    int64_t chunks = (numel + kRedChunk - 1) / kRedChunk;
    if (scratch_elems < chunks) {
        set_error("rf_mse: scratch of %lld doubles < %lld", (long long)scratch_elems, (long long)chunks);
        return RF_EWORKSPACE;
    }
    rf_sqdiff_partials<<<(unsigned)chunks, kRedThreads, 0, st>>>(a, b, numel, scratch);
    RF_TRY_LAUNCH("rf_sqdiff_partials");
    rf_sum_finish<<<1, 32, 0, st>>>(scratch, chunks, numel, out);
    RF_TRY_LAUNCH("rf_sum_finish");
    return RF_OK;
}
