// Bit-exact numpy keyed gaussian noise on sm_100a.
//
// Replaces NoiseSource.normal (reference latents.py:144-146), i.e.
//   np.random.Generator(np.random.Philox(key)).standard_normal(n)
// for many independent (key, n) draws in one batch.
//
// numpy's ziggurat consumes a data-dependent number of 64-bit words per output
// (1 on the fast path, 2 per wedge attempt, 1+2k for a k-iteration tail), so the
// stream offset of output i depends on every earlier output.  The GPU resolves it
// with a finite-state scan:
//   pass 1 (rf_zig_classify): every stream position p is classified independently
//     as if a draw started there -> len[p] (words consumed, following wedge
//     restarts) and val[p].  Position p acts on the state "distance to the next draw
//     start" s as  f_p(0) = len[p]-1, f_p(s) = s-1.  Each thread composes the maps of
//     its 16 positions into a 16-entry nibble table (states 0..15), a block scan
//     composes thread tables, and each block publishes its aggregate
//     (exit state, number of draw starts) for all 16 entry states.
//   pass 2 (rf_zig_scatter): a block folds the aggregates of the blocks before it
//     (draw start state 0 at position 0), then walks its positions and writes
//     out[rank] = val[p] for every draw start p with rank < n.
// A draw that needs more than RF_ZIG_MAX_LEN words (a >= 8-iteration tail loop,
// ~1e-12 per position) cannot be represented by the 16-state tables; pass 1 flags
// its draw and pass 2 resolves that draw with a sequential walk instead.
#include <math.h>
#include <math_constants.h>

#include "rf_common.cuh"
#include "rf_zig_tables.h"

namespace rf {

constexpr int kZigThreads = 256;
constexpr int kZigPerThread = 16;
constexpr int kZigBlock = kZigThreads * kZigPerThread;  // stream positions per block
constexpr int kZigMaxLen = 16;
constexpr int kMaxDrawsPerLaunch = 24;

struct DrawBatch {
    int count;
    int64_t block_off[kMaxDrawsPerLaunch + 1];  // first block of each draw
    int64_t pos_off[kMaxDrawsPerLaunch];         // first workspace position of each draw
    uint64_t k0[kMaxDrawsPerLaunch], k1[kMaxDrawsPerLaunch];
    int64_t n[kMaxDrawsPerLaunch];
    double *out[kMaxDrawsPerLaunch];
};

struct BlockAgg {
    uint64_t exit;      // nibble e = exit state for entry state e
    uint16_t cnt[16];   // draw starts inside the block for entry state e
};

__device__ __forceinline__ int nib(uint64_t t, int e) { return (int)((t >> (4 * e)) & 0xF); }

// (first a, then b)
__device__ __forceinline__ uint64_t compose(uint64_t a, uint64_t b) {
    uint64_t r = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) r |= (uint64_t)nib(b, nib(a, e)) << (4 * e);
    return r;
}

__device__ __forceinline__ int find_draw(const DrawBatch &B, int64_t blk) {
    int d = 0;
    while (d + 1 < B.count && B.block_off[d + 1] <= blk) ++d;
    return d;
}

struct ZigSmem {
    double wi[256];
    double fi[256];
    uint64_t ki[256];
};

__device__ __forceinline__ void load_zig(ZigSmem &z) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        z.wi[i] = rf_zig_wi[i];
        z.fi[i] = rf_zig_fi[i];
        z.ki[i] = rf_zig_ki[i];
    }
}

// log1p exactly as the reference's numpy computes it on this image's x86-64 hosts:
// numpy's npy_log1p is glibc 2.39's log1p, which the ifunc resolver dispatches to
// __log1p_fma on FMA/AVX2 CPUs -- the fdlibm algorithm (sysdeps/ieee754/dbl-64/
// s_log1p.c) compiled with FMA contraction.  The operation sequence below follows
// that object code (decoded from libm.so.6) one IEEE operation at a time, so the
// tail-path values of the ziggurat are bit-identical to numpy's.  CUDA's own log1p
// differs in the last ulp for ~0.5% of arguments.
__device__ __noinline__ double glibc_log1p_fma(double x) {
    const double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2, Lp3 = 0x1.2492494229359p-2;
    const double Lp4 = 0x1.c71c51d8e78afp-3, Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3;
    const double Lp7 = 0x1.2f112df3e5244p-3;
    const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
    const int hx = __double2hiint(x);
    const unsigned ax = (unsigned)hx & 0x7fffffffu;
    int k;
    double f, c = 0.0, u;
    unsigned hu;
    bool poly_k0 = false;
    if (hx <= 0x3fda8279) {                       // x < 0.41422 (all negatives too)
        if (ax > 0x3fefffffu) {                   // x <= -1
            if (x == -1.0) return -CUDART_INF;
            return CUDART_NAN;
        }
        if (ax <= 0x3e1fffffu) {                  // |x| < 2^-29
            if (ax > 0x3c8fffffu) return __fma_rn(-__dmul_rn(x, x), 0.5, x);
            return x;
        }
        if ((unsigned)hx + 0x402d413cu > 0x402d413cu) {  // -0.2929 < x < 0.41422: k = 0, f = x
            k = 0;
            f = x;
            hu = 1;
            poly_k0 = true;
        }
    } else if (hx > 0x7fefffff) {
        return __dadd_rn(x, x);
    }
    if (!poly_k0) {
        if (hx > 0x433fffff) {                    // x >= 2^53
            k = (hx >> 20) - 1023;
            u = x;
            c = 0.0;
            hu = (unsigned)hx;
        } else {
            u = __dadd_rn(x, 1.0);
            hu = (unsigned)__double2hiint(u);
            k = (int)(hu >> 20) - 1023;
            c = (k > 0) ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
            c = __ddiv_rn(c, u);
        }
        hu &= 0x000fffffu;
        if (hu > 0x6a09du) {
            k += 1;
            u = __hiloint2double((int)(hu | 0x3fe00000u), __double2loint(u));
            hu = (0x00100000u - hu) >> 2;
        } else {
            u = __hiloint2double((int)(hu | 0x3ff00000u), __double2loint(u));
        }
        f = __dsub_rn(u, 1.0);
    }
    const double hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
    if (hu == 0) {                                // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            const double kd = (double)k;
            return __fma_rn(kd, ln2_hi, __fma_rn(kd, ln2_lo, c));
        }
        const double R = __dmul_rn(__fma_rn(-f, 0x1.5555555555555p-1, 1.0), hfsq);
        if (k == 0) return __dsub_rn(f, R);
        const double kd = (double)k;
        const double t = __dsub_rn(__dsub_rn(R, __fma_rn(kd, ln2_lo, c)), f);
        return __fma_rn(kd, ln2_hi, -t);
    }
    const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
    const double z = __dmul_rn(s, s);
    const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
    const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
    double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
    R = __fma_rn(z4, R3, R);
    R = __fma_rn(z6, R4, R);
    const double w = __dmul_rn(__dadd_rn(R, hfsq), s);
    if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, w));
    const double kd = (double)k;
    const double t = __dsub_rn(__dsub_rn(hfsq, __dadd_rn(__fma_rn(kd, ln2_lo, c), w)), f);
    return __fma_rn(kd, ln2_hi, -t);
}

// A full draw starting at stream position p (numpy random_standard_normal, every
// branch).  Used for the 1-2% of positions that miss the fast path.
__device__ __noinline__ void zig_slow(uint64_t k0, uint64_t k1, uint64_t p, const ZigSmem &z,
                                      uint32_t *len_out, double *val_out) {
    uint64_t q = p;
    for (;;) {
        uint64_t r = philox_word(k0, k1, q);
        int idx = (int)(r & 0xff);
        r >>= 8;
        int sign = (int)(r & 1);
        uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = __dmul_rn((double)rabs, z.wi[idx]);
        if (sign) x = -x;
        if (rabs < z.ki[idx]) {
            *len_out = (uint32_t)(q + 1 - p);
            *val_out = x;
            return;
        }
        if (idx == 0) {
            uint64_t q2 = q + 1;
            for (;;) {
                double u1 = u64_to_unit_double(philox_word(k0, k1, q2));
                double u2 = u64_to_unit_double(philox_word(k0, k1, q2 + 1));
                q2 += 2;
                double xx = __dmul_rn(-RF_ZIG_NOR_INV_R, glibc_log1p_fma(-u1));
                double yy = -glibc_log1p_fma(-u2);
                if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
                    *len_out = (uint32_t)(q2 - p);
                    double m = __dadd_rn(RF_ZIG_NOR_R, xx);
                    *val_out = ((rabs >> 8) & 1) ? -m : m;
                    return;
                }
            }
        } else {
            double u = u64_to_unit_double(philox_word(k0, k1, q + 1));
            double lhs = __dadd_rn(__dmul_rn(__dsub_rn(z.fi[idx - 1], z.fi[idx]), u), z.fi[idx]);
            double rhs = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
            if (lhs < rhs) {
                *len_out = (uint32_t)(q + 2 - p);
                *val_out = x;
                return;
            }
            q += 2;
        }
    }
}

// ----------------------------------------------------------------- pass 1 --------
__global__ void __launch_bounds__(kZigThreads)
rf_zig_classify(const __grid_constant__ DrawBatch B, uint16_t *__restrict__ len_ws, double *__restrict__ val_ws,
                uint64_t *__restrict__ thread_tab, BlockAgg *__restrict__ aggs,
                int *__restrict__ long_flag) {
    __shared__ ZigSmem z;
    __shared__ uint64_t warp_tab[kZigThreads / 32];
    __shared__ uint64_t warp_cnt[kZigThreads / 32][4];
    load_zig(z);
    __syncthreads();

    const int64_t blk = blockIdx.x;
    const int d = find_draw(B, blk);
    const int64_t j = blk - B.block_off[d];
    const uint64_t k0 = B.k0[d], k1 = B.k1[d];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint64_t p0 = (uint64_t)j * kZigBlock + (uint64_t)t * kZigPerThread;
    const int64_t ws0 = B.pos_off[d] + (int64_t)j * kZigBlock + (int64_t)t * kZigPerThread;

    uint64_t tab = 0xFEDCBA9876543210ULL;  // identity
    uint64_t cnt_lo = 0, cnt_hi = 0;       // byte e = starts seen for entry state e
    bool any_long = false;
    uint16_t lens[kZigPerThread];
    double vals[kZigPerThread];
#pragma unroll
    for (int b = 0; b < kZigPerThread / 4; ++b) {
        uint64_t blk_ctr = ((p0 >> 2) + b) + 1;
        u64x4 w = philox4x64_10(blk_ctr, 0, 0, 0, k0, k1);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int q = b * 4 + i;
            uint64_t r = w.v[i];
            int idx = (int)(r & 0xff);
            uint64_t rr = r >> 8;
            uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
            double x = __dmul_rn((double)rabs, z.wi[idx]);
            if (rr & 1) x = -x;
            uint32_t len = 1;
            if (!(rabs < z.ki[idx])) zig_slow(k0, k1, p0 + q, z, &len, &x);
            if (len > kZigMaxLen) any_long = true;
            lens[q] = (uint16_t)(len > 0xFFFF ? 0xFFFF : len);
            vals[q] = x;
            // state map of this position applied after `tab`
            uint64_t tt = tab | (tab >> 1);
            tt |= tt >> 2;
            uint64_t zmask = ~tt & 0x1111111111111111ULL;  // nibbles equal to 0
            uint64_t lm1 = (uint64_t)((len - 1) > 15 ? 15 : (len - 1));
            tab = (tab - (0x1111111111111111ULL & ~zmask)) | (zmask * lm1);
            // count starts per entry state: spread nibble flags into byte lanes
            uint64_t lo = zmask & 0xFFFFFFFFULL, hi = zmask >> 32;
            lo = (lo | (lo << 16)) & 0x0000FFFF0000FFFFULL;
            lo = (lo | (lo << 8)) & 0x00FF00FF00FF00FFULL;
            lo = (lo | (lo << 4)) & 0x0F0F0F0F0F0F0F0FULL;
            hi = (hi | (hi << 16)) & 0x0000FFFF0000FFFFULL;
            hi = (hi | (hi << 8)) & 0x00FF00FF00FF00FFULL;
            hi = (hi | (hi << 4)) & 0x0F0F0F0F0F0F0F0FULL;
            cnt_lo += lo;
            cnt_hi += hi;
        }
    }
    // write classification
#pragma unroll
    for (int q = 0; q < kZigPerThread; ++q) {
        len_ws[ws0 + q] = lens[q];
        val_ws[ws0 + q] = vals[q];
    }
    if (any_long) atomicOr(long_flag + d, 1);

    // exclusive scan of thread tables (composition) within the block
    uint64_t incl = tab;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        uint64_t other = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl = compose(other, incl);
    }
    if (lane == 31) warp_tab[warp] = incl;
    __syncthreads();
    uint64_t warp_prefix = 0xFEDCBA9876543210ULL;
    for (int w = 0; w < warp; ++w) warp_prefix = compose(warp_prefix, warp_tab[w]);
    uint64_t lane_excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) lane_excl = 0xFEDCBA9876543210ULL;
    const uint64_t entry_tab = compose(warp_prefix, lane_excl);
    thread_tab[blk * kZigThreads + t] = entry_tab;

    // per-entry-state counts of the whole block: sum_t cnt_t[entry_tab(e)]
    uint64_t c4[4] = {0, 0, 0, 0};  // 16-bit lanes, entry e in word e/4, lane e%4
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        int s = nib(entry_tab, e);
        uint64_t c = s < 8 ? (cnt_lo >> (8 * s)) & 0xFF : (cnt_hi >> (8 * (s - 8))) & 0xFF;
        c4[e >> 2] += c << (16 * (e & 3));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) c4[k] += __shfl_xor_sync(0xffffffffu, c4[k], off);
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) warp_cnt[warp][k] = c4[k];
    }
    __syncthreads();
    if (t == 0) {
        uint64_t tot = 0xFEDCBA9876543210ULL;
        for (int w = 0; w < kZigThreads / 32; ++w) tot = compose(tot, warp_tab[w]);
        BlockAgg a;
        a.exit = tot;
        uint64_t s4[4] = {0, 0, 0, 0};
        for (int w = 0; w < kZigThreads / 32; ++w)
            for (int k = 0; k < 4; ++k) s4[k] += warp_cnt[w][k];
        for (int e = 0; e < 16; ++e) a.cnt[e] = (uint16_t)((s4[e >> 2] >> (16 * (e & 3))) & 0xFFFF);
        aggs[blk] = a;
    }
}

// ----------------------------------------------------------------- pass 2 --------
__global__ void __launch_bounds__(kZigThreads)
rf_zig_scatter(const __grid_constant__ DrawBatch B, const uint16_t *__restrict__ len_ws, const double *__restrict__ val_ws,
               const uint64_t *__restrict__ thread_tab, const BlockAgg *__restrict__ aggs,
               const int *__restrict__ long_flag, uint32_t *__restrict__ status) {
    __shared__ int s_entry;
    __shared__ long long s_base;
    __shared__ int warp_sum[kZigThreads / 32];
    const int64_t blk = blockIdx.x;
    const int d = find_draw(B, blk);
    const int64_t j = blk - B.block_off[d];
    const int64_t nblk = B.block_off[d + 1] - B.block_off[d];
    const int64_t n = B.n[d];
    double *out = B.out[d];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t wsd = B.pos_off[d];

    if (long_flag[d]) {
        // Sequential resolution of the whole draw (astronomically rare).
        if (j == 0 && t == 0) {
            int64_t p = 0, i = 0, m = nblk * kZigBlock;
            while (i < n && p < m) {
                out[i++] = val_ws[wsd + p];
                p += len_ws[wsd + p];
            }
            if (i < n) atomicOr(status, RF_STATUS_NOISE_SHORT);
            atomicOr(status, RF_STATUS_NOISE_LONG);
        }
        return;
    }
    if (t == 0) {
        int s = 0;
        long long base = 0;
        const BlockAgg *a = aggs + B.block_off[d];
        for (int64_t i = 0; i < j; ++i) {
            base += a[i].cnt[s];
            s = nib(a[i].exit, s);
        }
        s_entry = s;
        s_base = base;
        if (j == nblk - 1 && base + a[j].cnt[s] < n) atomicOr(status, RF_STATUS_NOISE_SHORT);
    }
    __syncthreads();
    const int64_t base = s_base;
    if (base >= n) return;
    int s = nib(thread_tab[blk * kZigThreads + t], s_entry);
    const int64_t ws0 = wsd + j * kZigBlock + (int64_t)t * kZigPerThread;
    uint16_t lens[kZigPerThread];
#pragma unroll
    for (int q = 0; q < kZigPerThread; ++q) lens[q] = len_ws[ws0 + q];
    uint32_t starts = 0;
    int c = 0;
#pragma unroll
    for (int q = 0; q < kZigPerThread; ++q) {
        if (s == 0) {
            starts |= 1u << q;
            ++c;
            s = lens[q] - 1;
        } else {
            --s;
        }
    }
    // block exclusive scan of c
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    int wp = 0;
    for (int w = 0; w < warp; ++w) wp += warp_sum[w];
    int64_t rank = base + wp + (incl - c);
#pragma unroll
    for (int q = 0; q < kZigPerThread; ++q) {
        if (starts & (1u << q)) {
            if (rank < n) out[rank] = val_ws[ws0 + q];
            ++rank;
        }
    }
}

__global__ void rf_uniform_kernel(const __grid_constant__ DrawBatch B) {
    const int64_t blk = blockIdx.x;
    const int d = find_draw(B, blk);
    const int64_t j = blk - B.block_off[d];
    const int64_t i = j * blockDim.x + threadIdx.x;
    if (i < B.n[d]) B.out[d][i] = u64_to_unit_double(philox_word(B.k0[d], B.k1[d], (uint64_t)i));
}

static int64_t draw_positions(int64_t n) {
    int64_t m = n + n / 16 + 1024;
    return (m + kZigBlock - 1) / kZigBlock * kZigBlock;
}

struct WsLayout {
    int64_t positions, blocks;
    int64_t off_len, off_val, off_tab, off_agg, off_flag, total;
};

static WsLayout layout(const rf_draw *draws, int count) {
    WsLayout L{};
    for (int i = 0; i < count; ++i) L.positions += draw_positions(draws[i].n);
    L.blocks = L.positions / kZigBlock;
    auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
    L.off_len = 0;
    L.off_val = al(L.off_len + L.positions * 2);
    L.off_tab = al(L.off_val + L.positions * 8);
    L.off_agg = al(L.off_tab + L.blocks * kZigThreads * 8);
    L.off_flag = al(L.off_agg + L.blocks * (int64_t)sizeof(BlockAgg));
    L.total = al(L.off_flag + kMaxDrawsPerLaunch * 4);
    return L;
}

}  // namespace rf

using namespace rf;

extern "C" int64_t rf_normal_workspace_bytes(const rf_draw *draws, int count) {
    // The batch is processed in chunks of kMaxDrawsPerLaunch draws reusing one
    // workspace, so the requirement is the largest chunk.
    int64_t best = 0;
    for (int c0 = 0; c0 < count; c0 += kMaxDrawsPerLaunch) {
        int c = count - c0 < kMaxDrawsPerLaunch ? count - c0 : kMaxDrawsPerLaunch;
        WsLayout L = layout(draws + c0, c);
        if (L.total > best) best = L.total;
    }
    return best;
}

extern "C" int rf_normal_fill(const rf_draw *draws, int count, void *workspace,
                              int64_t workspace_bytes, uint32_t *status, void *stream) {
    if (count < 0 || (count > 0 && (!draws || !workspace || !status))) {
        set_error("rf_normal_fill: null argument");
        return RF_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    for (int c0 = 0; c0 < count; c0 += kMaxDrawsPerLaunch) {
        int c = count - c0 < kMaxDrawsPerLaunch ? count - c0 : kMaxDrawsPerLaunch;
        const rf_draw *dr = draws + c0;
        WsLayout L = layout(dr, c);
        if (L.total > workspace_bytes) {
            set_error("rf_normal_fill: workspace %lld < %lld bytes", (long long)workspace_bytes,
                      (long long)L.total);
            return RF_EWORKSPACE;
        }
        DrawBatch B{};
        B.count = c;
        int64_t blk = 0, pos = 0;
        for (int i = 0; i < c; ++i) {
            if (dr[i].n < 0 || (dr[i].n > 0 && !dr[i].out)) {
                set_error("rf_normal_fill: bad draw %d", c0 + i);
                return RF_EINVAL;
            }
            B.block_off[i] = blk;
            B.pos_off[i] = pos;
            B.k0[i] = dr[i].k0;
            B.k1[i] = dr[i].k1;
            B.n[i] = dr[i].n;
            B.out[i] = dr[i].out;
            int64_t m = draw_positions(dr[i].n);
            pos += m;
            blk += m / kZigBlock;
        }
        B.block_off[c] = blk;
        char *ws = (char *)workspace;
        uint16_t *len_ws = (uint16_t *)(ws + L.off_len);
        double *val_ws = (double *)(ws + L.off_val);
        uint64_t *tab = (uint64_t *)(ws + L.off_tab);
        BlockAgg *aggs = (BlockAgg *)(ws + L.off_agg);
        int *flags = (int *)(ws + L.off_flag);
        RF_TRY_CUDA(cudaMemsetAsync(flags, 0, kMaxDrawsPerLaunch * sizeof(int), st));
        rf_zig_classify<<<(unsigned)blk, kZigThreads, 0, st>>>(B, len_ws, val_ws, tab, aggs, flags);
        RF_TRY_LAUNCH("rf_zig_classify");
        rf_zig_scatter<<<(unsigned)blk, kZigThreads, 0, st>>>(B, len_ws, val_ws, tab, aggs, flags,
                                                              status);
        RF_TRY_LAUNCH("rf_zig_scatter");
    }
    return RF_OK;
}

extern "C" int rf_uniform_fill(const rf_draw *draws, int count, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int threads = 256;
    for (int c0 = 0; c0 < count; c0 += kMaxDrawsPerLaunch) {
        int c = count - c0 < kMaxDrawsPerLaunch ? count - c0 : kMaxDrawsPerLaunch;
        DrawBatch B{};
        B.count = c;
        int64_t blk = 0;
        for (int i = 0; i < c; ++i) {
            const rf_draw &dd = draws[c0 + i];
            if (dd.n < 0 || (dd.n > 0 && !dd.out)) {
                set_error("rf_uniform_fill: bad draw %d", c0 + i);
                return RF_EINVAL;
            }
            B.block_off[i] = blk;
            B.k0[i] = dd.k0;
            B.k1[i] = dd.k1;
            B.n[i] = dd.n;
            B.out[i] = dd.out;
            blk += (dd.n + threads - 1) / threads;
        }
        B.block_off[c] = blk;
        if (blk == 0) continue;
        rf_uniform_kernel<<<(unsigned)blk, threads, 0, st>>>(B);
        RF_TRY_LAUNCH("rf_uniform_kernel");
    }
    return RF_OK;
}
