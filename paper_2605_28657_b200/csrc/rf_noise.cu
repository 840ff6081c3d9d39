// Bit-exact numpy keyed gaussian noise on sm_100a.
//
// Replaces NoiseSource.normal (reference latents.py:144-146), i.e.
//   np.random.Generator(np.random.Philox(key)).standard_normal(n)
// for many independent (key, n) draws in one batch.
//
// numpy's ziggurat consumes a data-dependent number of 64-bit words per output
// (1 on the fast path, 2 per wedge attempt, 1+2k for a k-iteration tail), so the
// stream offset of output i depends on every earlier output.  Two passes over the
// stream positions of every draw in the batch resolve it:
//   pass 1 (rf_zig_classify): one thread per Philox4x64-10 block (4 positions); every
//     position p is classified as if a draw started there -> len[p] (words consumed,
//     following wedge restarts) and val[p].  The slow paths read their extra words from
//     a register window (own block + the next thread's block, by shuffle).  Per block
//     of 512 positions the rare multi-word positions are compacted into a sorted list
//     that 16 lanes walk, one per entry state e (positions already consumed by the
//     previous block's last draw): the block aggregate (exit state, draw starts)[e].
//     The last block of a draw to finish (threadfence + counter) scans the draw's
//     aggregates from state 0 and publishes every block's entry state and output base.
//   pass 2 (rf_zig_scatter): each block re-walks its multi list with its entry state
//     and writes out[base + rank] = val[p] for every draw start p.
// A draw needing more than kZigMaxLen words (a >= 8-iteration tail loop, ~1e-12 per
// position) does not fit the 16-state tables; pass 1 flags it and pass 2 resolves that
// draw with a sequential walk instead.
#include <math.h>
#include <math_constants.h>

#include "rf_common.cuh"
#include "rf_zig_tables.h"

namespace rf {

constexpr int kZigThreads = 128;
constexpr int kZigPerThread = 4;   // one Philox4x64-10 block per thread
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

struct BlockEntry {
    int32_t state;      // positions of this block consumed by the previous draw
    int32_t pad;
    int64_t base;       // output index of this block's first draw start
};

struct DrawCtl {
    int32_t done;       // pass-1 blocks finished (last one scans)
    int32_t long_len;   // a draw needed > kZigMaxLen words
};

__device__ __forceinline__ int nib(uint64_t t, int e) { return (int)((t >> (4 * e)) & 0xF); }

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

// A full draw starting at window index q (numpy random_standard_normal, every branch),
// for the ~1.2% of positions that miss the fast path.  Words come from the 8-word
// register window `win` (valid for indices < nwin) and are recomputed past it.
struct Window {
    uint64_t w[8];
    int nwin;
    uint64_t base;  // stream position of w[0]
};

__device__ __forceinline__ uint64_t win_word(const Window &W, uint64_t k0, uint64_t k1, int i) {
    if (i < W.nwin) {
        uint64_t r = W.w[0];
#pragma unroll
        for (int k = 1; k < 8; ++k) r = i == k ? W.w[k] : r;
        return r;
    }
    return philox_word(k0, k1, W.base + (uint64_t)i);
}

__device__ __noinline__ void zig_slow(const Window &W, uint64_t k0, uint64_t k1, int q,
                                      const ZigSmem &z, uint32_t *len_out, double *val_out) {
    int qq = q;
    for (;;) {
        uint64_t r = win_word(W, k0, k1, qq);
        int idx = (int)(r & 0xff);
        r >>= 8;
        int sign = (int)(r & 1);
        uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = __dmul_rn((double)rabs, z.wi[idx]);
        if (sign) x = -x;
        if (rabs < z.ki[idx]) {
            *len_out = (uint32_t)(qq + 1 - q);
            *val_out = x;
            return;
        }
        if (idx == 0) {
            int q2 = qq + 1;
            for (;;) {
                double u1 = u64_to_unit_double(win_word(W, k0, k1, q2));
                double u2 = u64_to_unit_double(win_word(W, k0, k1, q2 + 1));
                q2 += 2;
                double xx = __dmul_rn(-RF_ZIG_NOR_INV_R, glibc_log1p_fma(-u1));
                double yy = -glibc_log1p_fma(-u2);
                if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
                    *len_out = (uint32_t)(q2 - q);
                    double m = __dadd_rn(RF_ZIG_NOR_R, xx);
                    *val_out = ((rabs >> 8) & 1) ? -m : m;
                    return;
                }
            }
        } else {
            double u = u64_to_unit_double(win_word(W, k0, k1, qq + 1));
            double lhs = __dadd_rn(__dmul_rn(__dsub_rn(z.fi[idx - 1], z.fi[idx]), u), z.fi[idx]);
            double rhs = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
            if (lhs < rhs) {
                *len_out = (uint32_t)(qq + 2 - q);
                *val_out = x;
                return;
            }
            qq += 2;
        }
    }
}

struct Multi {
    uint16_t pos;
    uint16_t len;
};

// Compact this block's multi-word positions (position-sorted) into smem; returns the count.
__device__ __forceinline__ int compact_multis(const uint16_t (&lens)[kZigPerThread], Multi *list,
                                              int *warp_tot) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int mine = 0;
#pragma unroll
    for (int q = 0; q < kZigPerThread; ++q) mine += lens[q] > 1;
    int incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int base = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kZigThreads / 32; ++w) {
        base += w < warp ? warp_tot[w] : 0;
        total += warp_tot[w];
    }
    int k = base + incl - mine;
#pragma unroll
    for (int q = 0; q < kZigPerThread; ++q) {
        if (lens[q] > 1) {
            list[k].pos = (uint16_t)(t * kZigPerThread + q);
            list[k].len = lens[q];
            ++k;
        }
    }
    __syncthreads();
    return total;
}

// Prefix of a draw's block aggregates from entry state 0, by the draw's last pass-1
// block: each thread composes a contiguous chunk into a 16-state (exit, count) table,
// a Kogge-Stone scan composes the chunk tables, and each thread then walks its chunk
// with its exact entry state, writing every block's (entry state, output base).
__device__ void draw_prefix(const BlockAgg *__restrict__ aggs, BlockEntry *__restrict__ entries,
                            int64_t nblk) {
    __shared__ uint64_t tex[2][kZigThreads];
    __shared__ uint32_t tcnt[2][kZigThreads][16];
    const int t = threadIdx.x;
    const int64_t ch = (nblk + kZigThreads - 1) / kZigThreads;
    const int64_t lo = t * ch, hi = lo + ch < nblk ? lo + ch : nblk;
    uint64_t ex = 0xFEDCBA9876543210ULL;
    uint32_t cnt[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) cnt[e] = 0;
    for (int64_t i = lo; i < hi; ++i) {
        const uint64_t bex = aggs[i].exit;
        uint64_t nex = 0;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int s = nib(ex, e);
            cnt[e] += aggs[i].cnt[s];
            nex |= (uint64_t)nib(bex, s) << (4 * e);
        }
        ex = nex;
    }
    int buf = 0;
    tex[buf][t] = ex;
#pragma unroll
    for (int e = 0; e < 16; ++e) tcnt[buf][t][e] = cnt[e];
    __syncthreads();
    // inclusive scan: table[t] = table[t - off] then table[t]
    for (int off = 1; off < kZigThreads; off <<= 1) {
        const int nb = buf ^ 1;
        if (t >= off) {
            const uint64_t aex = tex[buf][t - off], bex = tex[buf][t];
            uint64_t nex = 0;
            for (int e = 0; e < 16; ++e) {
                const int s = nib(aex, e);
                tcnt[nb][t][e] = tcnt[buf][t - off][e] + tcnt[buf][t][s];
                nex |= (uint64_t)nib(bex, s) << (4 * e);
            }
            tex[nb][t] = nex;
        } else {
            tex[nb][t] = tex[buf][t];
            for (int e = 0; e < 16; ++e) tcnt[nb][t][e] = tcnt[buf][t][e];
        }
        __syncthreads();
        buf = nb;
    }
    int s = 0;
    int64_t base = 0;
    if (t > 0) {
        s = nib(tex[buf][t - 1], 0);
        base = tcnt[buf][t - 1][0];
    }
    for (int64_t i = lo; i < hi; ++i) {
        entries[i].state = s;
        entries[i].base = base;
        base += aggs[i].cnt[s];
        s = nib(aggs[i].exit, s);
    }
}

// ----------------------------------------------------------------- pass 1 --------
__global__ void __launch_bounds__(kZigThreads)
rf_zig_classify(const __grid_constant__ DrawBatch B, uint16_t *__restrict__ len_ws,
                double *__restrict__ val_ws, BlockAgg *__restrict__ aggs,
                BlockEntry *__restrict__ entries, DrawCtl *__restrict__ ctl) {
    __shared__ ZigSmem z;
    __shared__ Multi list[kZigBlock];
    __shared__ int warp_tot[kZigThreads / 32];
    __shared__ int am_last;
    load_zig(z);
    __syncthreads();

    const int64_t blk = blockIdx.x;
    const int d = find_draw(B, blk);
    const int64_t j = blk - B.block_off[d];
    const uint64_t k0 = B.k0[d], k1 = B.k1[d];
    const int t = threadIdx.x, lane = t & 31;
    const uint64_t p0 = (uint64_t)j * kZigBlock + (uint64_t)t * kZigPerThread;
    const int64_t ws0 = B.pos_off[d] + (int64_t)j * kZigBlock + (int64_t)t * kZigPerThread;

    Window W;
    const u64x4 wv = philox4x64_10((p0 >> 2) + 1, 0, 0, 0, k0, k1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        W.w[i] = wv.v[i];
        W.w[4 + i] = __shfl_down_sync(0xffffffffu, wv.v[i], 1);
    }
    W.nwin = lane < 31 ? 8 : 4;
    W.base = p0;

    uint16_t lens[kZigPerThread];
    double vals[kZigPerThread];
    bool any_long = false;
#pragma unroll
    for (int q = 0; q < kZigPerThread; ++q) {
        const uint64_t r = W.w[q];
        const int idx = (int)(r & 0xff);
        const uint64_t rr = r >> 8;
        const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
        double x = __dmul_rn((double)rabs, z.wi[idx]);
        if (rr & 1) x = -x;
        uint32_t len = 1;
        if (!(rabs < z.ki[idx])) zig_slow(W, k0, k1, q, z, &len, &x);
        any_long |= len > kZigMaxLen;
        lens[q] = (uint16_t)(len > 0xFFFF ? 0xFFFF : len);
        vals[q] = x;
    }
    *reinterpret_cast<ushort4 *>(len_ws + ws0) = make_ushort4(lens[0], lens[1], lens[2], lens[3]);
    *reinterpret_cast<double2 *>(val_ws + ws0) = make_double2(vals[0], vals[1]);
    *reinterpret_cast<double2 *>(val_ws + ws0 + 2) = make_double2(vals[2], vals[3]);
    if (any_long) atomicOr(&ctl[d].long_len, 1);

    const int nm = compact_multis(lens, list, warp_tot);
    if (t < 16) {
        int covered_end = t, covered = t;
        for (int i = 0; i < nm; ++i) {
            const int p = list[i].pos;
            if (p >= covered_end) {
                const int end = p + list[i].len;
                covered += (end < kZigBlock ? end : kZigBlock) - (p + 1);
                covered_end = end;
            }
        }
        const int ex = covered_end > kZigBlock ? covered_end - kZigBlock : 0;
        uint64_t exmask = (uint64_t)(ex > 15 ? 15 : ex) << (4 * t);
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) exmask |= __shfl_xor_sync(0x0000ffffu, exmask, off);
        aggs[blk].cnt[t] = (uint16_t)(kZigBlock - covered);
        if (t == 0) aggs[blk].exit = exmask;
    }
    // last block of this draw to finish computes the draw's block prefix
    __threadfence();
    __syncthreads();
    const int64_t nblk = B.block_off[d + 1] - B.block_off[d];
    if (t == 0) am_last = atomicAdd(&ctl[d].done, 1) == (int)nblk - 1;
    __syncthreads();
    if (am_last) {
        __threadfence();
        draw_prefix(aggs + B.block_off[d], entries + B.block_off[d], nblk);
    }
}

// ----------------------------------------------------------------- pass 2 --------
__global__ void __launch_bounds__(kZigThreads)
rf_zig_scatter(const __grid_constant__ DrawBatch B, const uint16_t *__restrict__ len_ws,
               const double *__restrict__ val_ws, const BlockAgg *__restrict__ aggs,
               const BlockEntry *__restrict__ entries, const DrawCtl *__restrict__ ctl,
               uint32_t *__restrict__ status) {
    __shared__ int warp_tot[kZigThreads / 32];
    __shared__ Multi list[kZigBlock];
    __shared__ uint16_t cov_lo[kZigBlock], cov_hi[kZigBlock];
    __shared__ int n_cov;
    const int64_t blk = blockIdx.x;
    const int d = find_draw(B, blk);
    const int64_t j = blk - B.block_off[d];
    const int64_t nblk = B.block_off[d + 1] - B.block_off[d];
    const int64_t n = B.n[d];
    double *out = B.out[d];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t wsd = B.pos_off[d];

    if (ctl[d].long_len) {
        // Sequential resolution of the whole draw (a >= 8-iteration tail loop somewhere).
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
    const BlockEntry be = entries[blk];
    if (j == nblk - 1 && t == 0 && be.base + aggs[blk].cnt[be.state] < n)
        atomicOr(status, RF_STATUS_NOISE_SHORT);
    if (be.base >= n) return;
    const int64_t ws0 = wsd + j * kZigBlock + (int64_t)t * kZigPerThread;
    const ushort4 l4 = *reinterpret_cast<const ushort4 *>(len_ws + ws0);
    const uint16_t lens[kZigPerThread] = {l4.x, l4.y, l4.z, l4.w};
    const int nm = compact_multis(lens, list, warp_tot);
    if (t == 0) {
        int covered_end = be.state, k = 0;
        for (int i = 0; i < nm; ++i) {
            const int p = list[i].pos;
            if (p >= covered_end) {
                covered_end = p + list[i].len;
                cov_lo[k] = (uint16_t)(p + 1);
                cov_hi[k] = (uint16_t)(covered_end < kZigBlock ? covered_end : kZigBlock);
                ++k;
            }
        }
        n_cov = k;
    }
    __syncthreads();
    const int ncov = n_cov;
    uint32_t starts = 0;
    int c = 0;
#pragma unroll
    for (int q = 0; q < kZigPerThread; ++q) {
        const int p = t * kZigPerThread + q;
        bool cov = p < be.state;
        for (int i = 0; i < ncov && !cov; ++i) cov = p >= cov_lo[i] && p < cov_hi[i];
        if (!cov) {
            starts |= 1u << q;
            ++c;
        }
    }
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    __syncthreads();  // warp_tot reuse
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int wp = 0;
    for (int w2 = 0; w2 < warp; ++w2) wp += warp_tot[w2];
    int64_t rank = be.base + wp + (incl - c);
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
    int64_t off_len, off_val, off_agg, off_ent, off_ctl, total;
};

static WsLayout layout(const rf_draw *draws, int count) {
    WsLayout L{};
    for (int i = 0; i < count; ++i) L.positions += draw_positions(draws[i].n);
    L.blocks = L.positions / kZigBlock;
    auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
    L.off_len = 0;
    L.off_val = al(L.off_len + L.positions * 2);
    L.off_agg = al(L.off_val + L.positions * 8);
    L.off_ent = al(L.off_agg + L.blocks * (int64_t)sizeof(BlockAgg));
    L.off_ctl = al(L.off_ent + L.blocks * (int64_t)sizeof(BlockEntry));
    L.total = al(L.off_ctl + kMaxDrawsPerLaunch * (int64_t)sizeof(DrawCtl));
    return L;
}

}  // namespace rf

using namespace rf;

extern "C" int64_t rf_normal_workspace_bytes(const rf_draw *draws, int count) {
    // Chunks of kMaxDrawsPerLaunch draws reuse one workspace: size for the largest.
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
        BlockAgg *aggs = (BlockAgg *)(ws + L.off_agg);
        BlockEntry *ent = (BlockEntry *)(ws + L.off_ent);
        DrawCtl *ctl = (DrawCtl *)(ws + L.off_ctl);
        RF_TRY_CUDA(cudaMemsetAsync(ctl, 0, kMaxDrawsPerLaunch * sizeof(DrawCtl), st));
        rf_zig_classify<<<(unsigned)blk, kZigThreads, 0, st>>>(B, len_ws, val_ws, aggs, ent, ctl);
        RF_TRY_LAUNCH("rf_zig_classify");
        rf_zig_scatter<<<(unsigned)blk, kZigThreads, 0, st>>>(B, len_ws, val_ws, aggs, ent, ctl, status);
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
