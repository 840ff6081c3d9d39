// Shared device helpers for the ringflow B200 kernels (sm_100a).
#pragma once
#include <stdlib.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ringflow_b200.h"

namespace rf {

// ------------------------------------------------------------------ errors --------
void set_error(const char *fmt, ...);
int check_cuda(cudaError_t e, const char *what);
#define RF_TRY_CUDA(expr)                                         \
    do {                                                          \
        int _rc = ::rf::check_cuda((expr), #expr);                \
        if (_rc) return _rc;                                      \
    } while (0)
#define RF_TRY_LAUNCH(what)                                       \
    do {                                                          \
        int _rc = ::rf::check_cuda(cudaGetLastError(), what);     \
        if (_rc) return _rc;                                      \
    } while (0)

int sm_count();

// ------------------------------------------------- programmatic dependent launch ----
// Kernels of the DiT forward are launched with programmatic stream serialization: a
// kernel's CTAs may start (barrier init, TMEM alloc, descriptor prefetch) while the
// previous kernel drains, and block in pdl_wait() until its results are visible.  Every
// such kernel calls pdl_wait() before its first global-memory access and pdl_launch()
// right after, so at most two grids are in flight.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline int pdl_allowed() { return 1; }

// L2 residency window: while set (the DiT forward sets it to its fp32 residual stream),
// every kernel launched through launch_pdl / the GEMM launcher carries an access-policy
// window marking that range persisting in L2, so the residual stream read and rewritten
// by three epilogues per layer stays on chip instead of round-tripping through HBM.
struct L2Window {
    void *base = nullptr;
    size_t bytes = 0;
    float hit_ratio = 0.f;
};
inline thread_local L2Window g_l2_window;   // set per thread while a DiT forward is launched / captured

// appends the window attribute (if any) to at[n]; returns the new attribute count
inline unsigned add_l2_window(cudaLaunchAttribute *at, unsigned n) {
    if (!g_l2_window.base) return n;
    at[n].id = cudaLaunchAttributeAccessPolicyWindow;
    at[n].val.accessPolicyWindow.base_ptr = g_l2_window.base;
    at[n].val.accessPolicyWindow.num_bytes = g_l2_window.bytes;
    at[n].val.accessPolicyWindow.hitRatio = g_l2_window.hit_ratio;
    at[n].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[n].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    return n + 1;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
    cfg.attrs = at;
    cfg.numAttrs = add_l2_window(at, 1);
    return cudaLaunchKernelEx(&cfg, kern, static_cast<Args &&>(args)...);
}

// ------------------------------------------------------------------ philox --------
// Philox4x64-10 exactly as numpy's bit generator (numpy/random/src/philox/philox.h).
struct u64x4 {
    uint64_t v[4];
};

__device__ __forceinline__ u64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2,
                                               uint64_t c3, uint64_t k0, uint64_t k1) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
        uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += W0;
        k1 += W1;
    }
    u64x4 o;
    o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
    return o;
}

// Word p of the stream keyed (k0,k1): numpy increments the 256-bit counter before the
// first block, so position p lives in block counter (p/4 + 1), word p%4.
__device__ __forceinline__ uint64_t philox_word(uint64_t k0, uint64_t k1, uint64_t p) {
    uint64_t blk = (p >> 2) + 1;
    u64x4 o = philox4x64_10(blk, blk == 0 ? 1 : 0, 0, 0, k0, k1);
    return o.v[p & 3];
}

__device__ __forceinline__ double u64_to_unit_double(uint64_t w) {
    return __dmul_rn((double)(w >> 11), 1.0 / 9007199254740992.0);
}

}  // namespace rf
