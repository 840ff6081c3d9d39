// Windowed / full toy-codec decode on the tensor cores (reference
// codec.py:93-164): the dilated conv stack and the upsampler as implicit GEMMs on
// tcgen05 (kind::f16, fp32 accumulation in TMEM), quantize_pcm fused into the epilogue.
//
// Precision.  Every operand is an unevaluated sum of two fp16 values, x = hi + lo with
// hi = fp16(x), lo = fp16(x - hi) (22-bit significand), and each product is expanded as
// hi*Whi + hi*Wlo + lo*Whi (three MMAs, the lo*lo term ~2^-22 dropped), accumulated in
// fp32.  The result is within ~1e-6 relative of the float64 reference before quantize,
// i.e. within 1 LSB of its int16 samples (1 LSB = 3e-5 of full scale).  Latent values
// beyond fp16's range (|x| > 65504, ~10^4 times the pipeline's latents) are clamped to it.
// tanh and quantize_pcm run in fp32 on the fp32 accumulator.
//
// Tiles.  A CTA owns 128 consecutive extended frames (M = 128 rows of every MMA):
// rows i <-> global frame gbase + i, gbase = first output frame - rf.  Layer l computes all
// 128 rows; row i of layer l is exact while its receptive field stays inside the tile, so
// after L layers rows [rf, 128 - rf) hold exact activations: P = 128 - 2 rf output frames
// per tile (98 at rf = 15).  Rows outside the valid range [vlo, vhi) are zero at the input
// and after every layer (the reference's padding and re-zeroing, codec.py:104-112).
// Because every row's arithmetic is the same whatever the tile, windowed == full holds bit
// for bit on the GPU whenever overlap >= rf, as in the reference's contract.
//
// Dilated conv without im2col.  Activations live in shared memory in the canonical
// no-swizzle K-major layout with 8-row core matrices packed row-contiguously
// ([k/8][row][8] halves, 16 B per row per k-chunk, SBO = 128 B): row r of k-chunk j sits
// at j * LBO + 16 r, so the operand for tap t (rows shifted by (t - 1) d) is the same
// buffer with the descriptor's start address moved by 16 (t - 1) d bytes.  The three taps
// are three accumulating MMA groups into one TMEM accumulator; the epilogue (tanh, mask,
// hi/lo split) writes the next layer's operand in place.
//
// Upsampler.  pcm[f][j] = quantize(sum_c h[f][c] U[j][c]): the hop columns are cut into
// chunks of cw <= 128 (N of the MMA); a CTA owns a slice of the chunks of its tile (the
// grid is tiles x slices, sized to the SM count), double-buffers them in TMEM (2 x 256
// columns) so the quantize epilogue of chunk c overlaps the MMAs of chunk c+1, and writes
// each row's int16 piece with a bulk (TMA) store from shared memory.
//
// Roles (576 threads): warps 0-15 epilogue (warp w: TMEM lanes 32 (w % 4) .. +31, column
// group w / 4), warp 16 weight producer (1-D bulk copies of pre-packed weight blocks into a
// 2-slot ring), warp 17 MMA issuer.  The epilogue is bound by the SM's conversion / MUFU
// unit (16 results per clock): tanh uses one MUFU op (ex2) with the reciprocal refined on
// the FMA pipe, and the fp16 splits use packed conversions.
#include <cuda_fp16.h>
#include <math.h>

#include "rf_common.cuh"
#include "rf_sm100.cuh"

namespace rf::dtc {
using namespace ::rf::sm100;

constexpr int kRows = 128;           // M of every MMA
constexpr int kPad = 16;             // zero rows above / below the tile (max dilation)
constexpr int kBufRows = kRows + 2 * kPad;
// upsampler chunk width (N): 128 -- hop 1920 in 15 chunks, one per CTA of a 3-s window
// (was 240: 8 chunks; the window's upsampler phase 3.4 -> 2.5 us, tools/decode_trace.py)
constexpr int kMaxCW = 128;
constexpr int kEpiWarps = 16;         // 4 column groups x 4 lane quarters
constexpr int kGroups = kEpiWarps / 4;
constexpr int kThreads = (kEpiWarps + 2) * 32;
constexpr int kMaxRF = 56;           // P = 128 - 2 rf >= 16

struct Args {
    const double *latent;     // [frames, C]
    int64_t frames;
    int C;
    const uint8_t *packed;    // rf_decode_tc_pack layout
    int32_t dil[RF_MAX_CODEC_LAYERS];
    int L, rf;
    int64_t vlo, vhi;         // valid global frame range
    int64_t start, nout;      // output frames [start, start + nout)
    int64_t hop;
    int cw, nch;              // chunk width, chunks per frame
    int slices;               // column slices per tile (grid = tiles x slices)
    int16_t *out;             // [nout * hop]
    unsigned long long *trace;   // debugging: globaltimer stamps [cta][32] (null in production)
};
__device__ __forceinline__ void dtrace(const Args &A, int slot) {
    if (A.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        A.trace[blockIdx.x * 32 + slot] = t;
    }
}

__host__ __device__ constexpr uint32_t conv_bytes(int CP) { return 3u * 2u * CP * CP * 2u; }
__host__ __device__ constexpr uint32_t chunk_bytes(int CP, int cw) { return 2u * CP * cw * 2u; }
__host__ __device__ constexpr uint32_t stage_row_bytes(int cw) {
    // row stride of the output staging buffer: 16-byte multiple, odd in 16-byte units
    // (a warp's 32 row writes then spread over all banks)
    return ((cw * 2 + 15) / 16 % 2 == 0) ? (cw * 2 + 15) / 16 * 16 + 16 : (cw * 2 + 15) / 16 * 16;
}
template <int CP>
struct Smem {
    // [CP/8][kBufRows (+1 pad row)][8] halves: k-chunks (kBufRows + 1) * 16 B apart, so the
    // 8 k-chunks of one row fall on different banks
    static constexpr uint32_t LBO_A = (kBufRows + 1) * 16;
    static constexpr uint32_t ACT_PIECE = (CP / 8) * LBO_A;
    static constexpr uint32_t SLOT = conv_bytes(CP) > chunk_bytes(CP, kMaxCW) ? conv_bytes(CP)
                                                                              : chunk_bytes(CP, kMaxCW);
    static constexpr uint32_t ACT = 0;
    static constexpr uint32_t RING = ACT + 2 * ACT_PIECE;
    static constexpr uint32_t STAGE = RING + 2 * SLOT;
    static constexpr uint32_t BARS = STAGE + kRows * stage_row_bytes(kMaxCW);
    static constexpr uint32_t TOTAL = BARS + 16 * 8 + 16;
};

// no-swizzle K-major operand: 8-row core matrices 128 B apart (SBO), k-chunks lbo apart
__device__ __forceinline__ uint64_t sdesc_interleave(uint32_t saddr, uint32_t lbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
}
// kind::f16 with fp16 A and B, fp32 D, both K-major
__device__ __forceinline__ uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint32_t pack_half2(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}
// 8 values -> (hi, lo) fp16 pieces, 16 B each (packed conversions: F2FP on the ALU pipe,
// not the quarter-rate single-value F2F)
__device__ __forceinline__ void split8(const float (&v)[8], uint4 &hi, uint4 &lo) {
    uint32_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __half2 a = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        const float2 af = __half22float2(a);
        const __half2 b = __floats2half2_rn(v[2 * i] - af.x, v[2 * i + 1] - af.y);
        h[i] = *reinterpret_cast<const uint32_t *>(&a);
        l[i] = *reinterpret_cast<const uint32_t *>(&b);
    }
    hi = make_uint4(h[0], h[1], h[2], h[3]);
    lo = make_uint4(l[0], l[1], l[2], l[3]);
}
// quantize_pcm (codec.py:27-31): copysign(floor(|32767 x| + 0.5), x) clipped to int16 --
// the truncating conversion of +-(|s| + 0.5) with saturation (fp32; the +-0.5 rounding of
// s = 32767 x is where a 1-LSB difference from the float64 reference can arise)
__device__ __forceinline__ uint32_t quantize2(float x0, float x1) {
    const float s0 = x0 * 32767.f, s1 = x1 * 32767.f;
    const float t0 = copysignf(fabsf(s0) + 0.5f, s0), t1 = copysignf(fabsf(s1) + 0.5f, s1);
    int16_t q0, q1;
    asm("cvt.rzi.sat.s16.f32 %0, %1;" : "=h"(q0) : "f"(t0));
    asm("cvt.rzi.sat.s16.f32 %0, %1;" : "=h"(q1) : "f"(t1));
    return (uint32_t)(uint16_t)q0 | ((uint32_t)(uint16_t)q1 << 16);
}
// tanh(x) = 1 - 2 / (e^{2x} + 1) with one MUFU op (ex2) and the reciprocal by Newton steps
// on the FMA pipe (the MUFU unit, 16 / clk / SM, would bound this epilogue otherwise):
// absolute error ~1e-7, which is what reaches the output (the next operand keeps 22 bits).
// Two values at a time on the packed fp32 pipe (FFMA2 / FMUL2, sm_100): the conv epilogue
// is issue-bound, and the pair form halves its FMA-pipe instructions (1.45 -> 1.1 us per
// layer of the 3-s window decode, tools/decode_trace.py).
__device__ __forceinline__ uint64_t pack_f2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 unpack_f2(uint64_t r) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
    return make_float2(a, b);
}
__device__ __forceinline__ float2 tanh_abs2(float x0, float x1) {
    x0 = fminf(fmaxf(x0, -9.f), 9.f);
    x1 = fminf(fmaxf(x1, -9.f), 9.f);
    const float d0 = __expf(2.f * x0) + 1.f, d1 = __expf(2.f * x1) + 1.f;
    uint64_t d = pack_f2(d0, d1), r = pack_f2(__uint_as_float(0x7EF311C3u - __float_as_uint(d0)),
                                              __uint_as_float(0x7EF311C3u - __float_as_uint(d1)));
    const uint64_t two = pack_f2(2.f, 2.f);
#pragma unroll
    for (int i = 0; i < 3; ++i) {   // r = r * (2 - d * r)
        uint64_t t;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(d ^ 0x8000000080000000ull), "l"(r), "l"(two));
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(r), "l"(t));
    }
    uint64_t y;   // 1 - 2 r
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(y) : "l"(r), "l"(pack_f2(-2.f, -2.f)), "l"(pack_f2(1.f, 1.f)));
    return unpack_f2(y);
}

template <int CP>
__global__ void __launch_bounds__(kThreads, 1) rf_decode_tc_kernel(const __grid_constant__ Args A) {
    using S = Smem<CP>;
    constexpr int KC8 = CP / 8;          // 16-byte k-chunks per row
    constexpr uint32_t LBO_A = S::LBO_A;
    constexpr uint32_t LBO_W = CP * 16;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S::BARS);
    uint64_t *full = bars + 0;        // [2] weight slot loaded
    uint64_t *empty = bars + 2;       // [2] weight slot consumed
    uint64_t *act_ready = bars + 4;   // next operand written (256 arrivals)
    uint64_t *conv_full = bars + 5;   // conv accumulator ready
    uint64_t *ufull = bars + 6;       // [2] upsampler accumulator ready
    uint64_t *tmem_empty = bars + 8;  // [2] upsampler accumulator drained (256 arrivals)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 10);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t tile = blockIdx.x / A.slices;
    const int slice = blockIdx.x % A.slices;
    const int P = kRows - 2 * A.rf;
    const int64_t g0 = A.start + tile * P;        // first output frame of the tile
    const int64_t gbase = g0 - A.rf;              // frame of row 0
    const int c_begin = (int)((int64_t)slice * A.nch / A.slices);
    const int c_end = (int)((int64_t)(slice + 1) * A.nch / A.slices);
    const uint8_t *wconv = A.packed;
    const uint8_t *wup = A.packed + (size_t)A.L * conv_bytes(CP);
    const uint32_t chunk_b = chunk_bytes(CP, A.cw);

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
            mbar_init(&ufull[i], 1);
            mbar_init(&tmem_empty[i], kEpiWarps);   // one arrival per epilogue warp
        }
        mbar_init(act_ready, kEpiWarps);
        mbar_init(conv_full, 1);
        mbar_fence_init();
    }
    if (threadIdx.x == 0) dtrace(A, 0);
    if (warp == kEpiWarps + 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // programmatic dependent launch: the barrier / TMEM setup above overlaps the previous
    // kernel's tail; the latent and the weights are read only after it has completed
    pdl_wait();
    pdl_launch();
    if (threadIdx.x == 0) dtrace(A, 1);

    if (warp == kEpiWarps) {
        // ---------------------------------------------------------- weight producer
        if (lane == 0) {
            const int nblk = A.L + (c_end - c_begin);
            for (int b = 0; b < nblk; ++b) {
                const int slot = b & 1, use = b >> 1;
                mbar_wait(&empty[slot], (use & 1) ^ 1);
                const uint32_t dst = sbase + S::RING + slot * S::SLOT;
                const bool conv = b < A.L;
                const uint32_t bytes = conv ? conv_bytes(CP) : chunk_b;
                const uint8_t *src = conv ? wconv + (size_t)b * conv_bytes(CP)
                                          : wup + (size_t)(c_begin + b - A.L) * chunk_b;
                mbar_expect_tx(&full[slot], bytes);
                bulk_g2s(dst, src, bytes, &full[slot]);
            }
        }
    } else if (warp == kEpiWarps + 1) {
        // ---------------------------------------------------------------- MMA issuer
        if (lane == 0) {
            const uint32_t act_hi = sbase + S::ACT, act_lo = act_hi + S::ACT_PIECE;
            int blk = 0;
            for (int l = 0; l < A.L; ++l, ++blk) {
                const int slot = blk & 1, use = blk >> 1;
                mbar_wait(act_ready, l & 1);
                dtrace(A, 2 + 2 * l);          // operand of layer l ready
                mbar_wait(&full[slot], use & 1);
                dtrace(A, 3 + 2 * l);          // weights of layer l ready
                tc_fence_after();
                const uint32_t w = sbase + S::RING + slot * S::SLOT;
                const uint32_t idesc = idesc_f16(kRows, CP);
                const int d = A.dil[l];
                uint32_t acc = 0;
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    const uint32_t row0 = (uint32_t)(kPad + (t - 1) * d) * 16u;
                    const uint32_t w_hi = w + (2 * t) * (CP * CP * 2), w_lo = w_hi + CP * CP * 2;
#pragma unroll
                    for (int kc = 0; kc < CP / 16; ++kc) {
                        const uint64_t ah = sdesc_interleave(act_hi + 2 * kc * LBO_A + row0, LBO_A);
                        const uint64_t al = sdesc_interleave(act_lo + 2 * kc * LBO_A + row0, LBO_A);
                        const uint64_t bh = sdesc_interleave(w_hi + 2 * kc * LBO_W, LBO_W);
                        const uint64_t bl = sdesc_interleave(w_lo + 2 * kc * LBO_W, LBO_W);
                        umma_bf16(tmem, ah, bh, idesc, acc);
                        umma_bf16(tmem, ah, bl, idesc, 1u);
                        umma_bf16(tmem, al, bh, idesc, 1u);
                        acc = 1u;
                    }
                }
                umma_commit(&empty[slot]);
                umma_commit(conv_full);
            }
            // upsampler chunks
            mbar_wait(act_ready, A.L & 1);
            dtrace(A, 12);
            tc_fence_after();
            const uint32_t lbo_u = (uint32_t)A.cw * 16u;
            for (int c = c_begin; c < c_end; ++c, ++blk) {
                const int j = c - c_begin, buf = j & 1, ub = j >> 1;
                const int slot = blk & 1, use = blk >> 1;
                const int n = (int)(A.hop - (int64_t)c * A.cw < A.cw ? A.hop - (int64_t)c * A.cw : A.cw);
                mbar_wait(&tmem_empty[buf], (ub & 1) ^ 1);
                mbar_wait(&full[slot], use & 1);
                if (j < 4) dtrace(A, 13 + j);   // chunk weights ready
                tc_fence_after();
                const uint32_t u_hi = sbase + S::RING + slot * S::SLOT;
                const uint32_t u_lo = u_hi + (uint32_t)CP * A.cw * 2u;
                const uint32_t idesc = idesc_f16(kRows, n);
                const uint32_t d_tmem = tmem + buf * 256;
#pragma unroll
                for (int kc = 0; kc < CP / 16; ++kc) {
                    const uint32_t arow = (uint32_t)kPad * 16u;
                    const uint64_t ah = sdesc_interleave(act_hi + 2 * kc * LBO_A + arow, LBO_A);
                    const uint64_t al = sdesc_interleave(act_lo + 2 * kc * LBO_A + arow, LBO_A);
                    const uint64_t bh = sdesc_interleave(u_hi + 2 * kc * lbo_u, lbo_u);
                    const uint64_t bl = sdesc_interleave(u_lo + 2 * kc * lbo_u, lbo_u);
                    umma_bf16(d_tmem, ah, bh, idesc, kc > 0 ? 1u : 0u);
                    umma_bf16(d_tmem, ah, bl, idesc, 1u);
                    umma_bf16(d_tmem, al, bh, idesc, 1u);
                }
                umma_commit(&empty[slot]);
                umma_commit(&ufull[buf]);
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue
        const int q = warp & 3, grp = warp >> 2;
        const int row = q * 32 + lane;                       // tile row = TMEM lane
        const int64_t g = gbase + row;
        const bool valid = g >= A.vlo && g < A.vhi;
        const uint32_t act_hi = sbase + S::ACT, act_lo = act_hi + S::ACT_PIECE;
        const int et = threadIdx.x;                          // 0 .. 511
        // zero the pad rows (read by the shifted taps), both pieces
        for (int i = et; i < 2 * KC8 * 2 * kPad; i += kEpiWarps * 32) {
            const int piece = i / (KC8 * 2 * kPad), r = i % (KC8 * 2 * kPad);
            const int kc = r / (2 * kPad), pr = r % (2 * kPad);
            const int brow = pr < kPad ? pr : kBufRows - 2 * kPad + pr;
            st_shared_v4((piece ? act_lo : act_hi) + kc * LBO_A + brow * 16, make_uint4(0, 0, 0, 0));
        }
        // layer-0 operand: the latent rows (zero outside the valid range), split hi / lo;
        // each thread's row chunks are loaded before any is converted (one round trip)
        constexpr int kItems = (kRows * KC8 + kEpiWarps * 32 - 1) / (kEpiWarps * 32);   // per thread
        double x[kItems][8];
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
            const int i = et + it * kEpiWarps * 32;
            if (i >= kRows * KC8) break;
            const int r = i % kRows, kc = i / kRows;
            const int64_t gr = gbase + r;
            const bool in = gr >= A.vlo && gr < A.vhi;
            if (in && (A.C % 8) == 0) {
                const double2 *src = reinterpret_cast<const double2 *>(A.latent + gr * A.C + kc * 8);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double2 d2 = kc * 8 < A.C ? __ldg(src + e) : make_double2(0.0, 0.0);
                    x[it][2 * e] = d2.x;
                    x[it][2 * e + 1] = d2.y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int c = kc * 8 + e;
                    x[it][e] = (in && c < A.C) ? A.latent[gr * A.C + c] : 0.0;
                }
            }
        }
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
            const int i = et + it * kEpiWarps * 32;
            if (i >= kRows * KC8) break;
            const int r = i % kRows, kc = i / kRows;
            __half xh[8], xl[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                // one fp64 -> fp32 conversion, then the hi / lo split in fp32 (exact: f - hi
                // is representable), as the activations are split -- fp64 ops are the slow ones
                const float f = fminf(fmaxf((float)x[it][e], -65504.f), 65504.f);
                xh[e] = __float2half_rn(f);
                xl[e] = __float2half_rn(f - __half2float(xh[e]));
            }
            uint32_t h[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                h[e] = pack_half2(xh[2 * e], xh[2 * e + 1]);
                lw[e] = pack_half2(xl[2 * e], xl[2 * e + 1]);
            }
            st_shared_v4(act_hi + kc * LBO_A + (kPad + r) * 16, make_uint4(h[0], h[1], h[2], h[3]));
            st_shared_v4(act_lo + kc * LBO_A + (kPad + r) * 16, make_uint4(lw[0], lw[1], lw[2], lw[3]));
        }
        fence_proxy_async_smem();
        if (threadIdx.x == 0) dtrace(A, 17);   // latent operand written (thread 0's part)
        __syncwarp();
        if (lane == 0) mbar_arrive(act_ready);   // per warp: 16 arrivals, not 512
        // conv layers: tanh, mask, split into the next operand (in place)
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        for (int l = 0; l < A.L; ++l) {
            mbar_wait(conv_full, l & 1);
            if (threadIdx.x == 0) dtrace(A, 18 + l);   // accumulator of layer l ready
            tc_fence_after();
            constexpr int KPG = (KC8 + kGroups - 1) / kGroups;   // k-chunks per column group
            float v[KPG][8];
#pragma unroll
            for (int kk = 0; kk < KPG; ++kk)
                if (grp + kk * kGroups < KC8) tmem_ld8(lane_base + (grp + kk * kGroups) * 8, v[kk]);
            tmem_ld_wait();
            for (int kk = 0; kk < KPG; ++kk) {
                const int kc = grp + kk * kGroups;
                if (kc >= KC8) break;
                if (valid) {
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        const float2 y = tanh_abs2(v[kk][e], v[kk][e + 1]);
                        v[kk][e] = y.x;
                        v[kk][e + 1] = y.y;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) v[kk][e] = 0.f;
                }
                uint4 hi, lo;
                split8(v[kk], hi, lo);
                st_shared_v4(act_hi + kc * LBO_A + (kPad + row) * 16, hi);
                st_shared_v4(act_lo + kc * LBO_A + (kPad + row) * 16, lo);
            }
            tc_fence_before();
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(act_ready);
        }
        // upsampler chunks: quantize, stage the row's piece, bulk-store it
        const bool out_row = row >= A.rf && row < A.rf + P && g < A.start + A.nout;
        const uint32_t srow = sbase + S::STAGE + row * stage_row_bytes(A.cw);
        // column group grp owns 8-column units [u0, u1) of every chunk
        const int n8c = A.cw / 8;
        const int u0 = grp * n8c / kGroups, u1 = (grp + 1) * n8c / kGroups;
        for (int c = c_begin; c < c_end; ++c) {
            const int j = c - c_begin, buf = j & 1, ub = j >> 1;
            mbar_wait(&ufull[buf], ub & 1);
            tc_fence_after();
            bulk_wait_read0();                                  // this row's previous store
            const int64_t col0 = (int64_t)c * A.cw + u0 * 8;
            int64_t ncols = A.hop - col0 < (u1 - u0) * 8 ? A.hop - col0 : (u1 - u0) * 8;
            if (ncols < 0) ncols = 0;
            const uint32_t taddr = lane_base + buf * 256;
            for (int k8 = u0; k8 < u1; k8 += 4) {   // 4 loads in flight per wait
                float v[4][8];
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (k8 + b < u1) tmem_ld8(taddr + (k8 + b) * 8, v[b]);
                tmem_ld_wait();
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if (k8 + b >= u1) break;
                    uint32_t p[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) p[e] = quantize2(v[b][2 * e], v[b][2 * e + 1]);
                    st_shared_v4(srow + (k8 + b) * 16, make_uint4(p[0], p[1], p[2], p[3]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[buf]);
            fence_proxy_async_smem();
            if (out_row && ncols > 0) {
                int16_t *dst = A.out + (g - A.start) * A.hop + col0;
                bulk_s2g(dst, srow + u0 * 16, (uint32_t)ncols * 2u);
                bulk_commit();
            }
        }
        // the staging buffer must stay until the stores have READ it; their global writes
        // complete before the kernel does
        bulk_wait_read0();
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) dtrace(A, 31);
    if (warp == kEpiWarps + 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

static unsigned long long *g_dtrace = nullptr;   // debugging timeline (rf_decode_set_trace)

// weights -> (hi, lo) fp16 blocks in the kernel's shared-memory operand layouts:
//   conv layer l: [tap][piece][k/8][n = out channel][8]   (B[n][k] = kernels[l][tap][k][n])
//   upsampler chunk ch: [piece][k/8][n = sample ch*cw + n][8]   (B[n][k] = U[j][k] = upT[k][j])
// zero for padded channels / samples beyond hop
__global__ void rf_decode_tc_pack_kernel(const double *kernels, int L, int C, int CP, const double *upT,
                                         int64_t hop, int cw, int nch, __half *out) {
    const int64_t conv_elems = (int64_t)L * 3 * 2 * CP * CP;
    const int64_t up_elems = (int64_t)nch * 2 * CP * cw;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < conv_elems + up_elems;
         i += (int64_t)gridDim.x * blockDim.x) {
        double w;
        int piece;
        if (i < conv_elems) {
            int64_t r = i;
            const int e = (int)(r % 8); r /= 8;
            const int n = (int)(r % CP); r /= CP;
            const int kc = (int)(r % (CP / 8)); r /= CP / 8;
            piece = (int)(r % 2); r /= 2;
            const int t = (int)(r % 3);
            const int l = (int)(r / 3);
            const int k = kc * 8 + e;
            w = (k < C && n < C) ? kernels[(((int64_t)l * 3 + t) * C + k) * C + n] : 0.0;
        } else {
            int64_t r = i - conv_elems;
            const int e = (int)(r % 8); r /= 8;
            const int n = (int)(r % cw); r /= cw;
            const int kc = (int)(r % (CP / 8)); r /= CP / 8;
            piece = (int)(r % 2);
            const int64_t ch = r / 2;
            const int k = kc * 8 + e;
            const int64_t jj = ch * cw + n;
            w = (k < C && jj < hop) ? upT[(int64_t)k * hop + jj] : 0.0;
        }
        const __half hi = __double2half(w);
        out[i] = piece == 0 ? hi : __double2half(w - (double)__half2float(hi));
    }
}

struct Geometry {
    int CP, cw, nch;
    int64_t bytes;
};
inline bool geometry(int64_t C, int64_t hop, int32_t L, Geometry &g) {
    if (C < 1 || C > 64 || hop < 16 || hop % 16 != 0 || L < 1 || L > RF_MAX_CODEC_LAYERS) return false;
    g.CP = (int)((C + 15) / 16 * 16);
    g.nch = (int)((hop + kMaxCW - 1) / kMaxCW);
    g.cw = (int)(((hop + g.nch - 1) / g.nch + 15) / 16 * 16);
    g.bytes = (int64_t)L * conv_bytes(g.CP) + (int64_t)g.nch * chunk_bytes(g.CP, g.cw);
    return true;
}

}  // namespace rf::dtc

using namespace rf;

extern "C" int64_t rf_decode_tc_packed_bytes(int64_t channels, int64_t hop, int32_t n_layers) {
    dtc::Geometry g;
    return dtc::geometry(channels, hop, n_layers, g) ? g.bytes : 0;
}

extern "C" int rf_decode_tc_pack(const double *kernels, int32_t n_layers, int64_t channels, const double *upsample_t,
                                 int64_t hop, void *packed, int64_t packed_bytes, void *stream) {
    dtc::Geometry g;
    if (!kernels || !upsample_t || !packed || !dtc::geometry(channels, hop, n_layers, g)) {
        set_error("rf_decode_tc_pack: unsupported shape (C=%lld, hop=%lld, L=%d) or null argument",
                  (long long)channels, (long long)hop, n_layers);
        return RF_EINVAL;
    }
    if (packed_bytes < g.bytes || ((uintptr_t)packed & 15)) {
        set_error("rf_decode_tc_pack: packed buffer too small or misaligned (%lld < %lld)",
                  (long long)packed_bytes, (long long)g.bytes);
        return RF_EINVAL;
    }
    dtc::rf_decode_tc_pack_kernel<<<296, 256, 0, (cudaStream_t)stream>>>(
        kernels, n_layers, (int)channels, g.CP, upsample_t, hop, g.cw, g.nch, (__half *)packed);
    RF_TRY_LAUNCH("rf_decode_tc_pack_kernel");
    return RF_OK;
}

extern "C" int rf_decode_window_tc(const double *latent, int64_t frames, int64_t channels, const void *packed,
                                   const int32_t *dilations, int32_t n_layers, int64_t hop, int64_t start,
                                   int64_t stop, int64_t overlap, int32_t full, int16_t *out, void *stream) {
    using namespace rf::dtc;
    Geometry g;
    if (!latent || !packed || !dilations || !out) {
        set_error("rf_decode_window_tc: null argument");
        return RF_EINVAL;
    }
    if (!geometry(channels, hop, n_layers, g)) {
        set_error("rf_decode_window_tc: unsupported shape (C=%lld must be in [1, 64], hop=%lld a multiple of 16, L=%d)",
                  (long long)channels, (long long)hop, n_layers);
        return RF_EINVAL;
    }
    if (!(0 <= start && start < stop && stop <= frames) || overlap < 0) {
        set_error("rf_decode_window_tc: window (%lld, %lld) outside [0, %lld)", (long long)start, (long long)stop,
                  (long long)frames);
        return RF_EINVAL;
    }
    if (((uintptr_t)out & 15) || ((uintptr_t)packed & 15)) {
        set_error("rf_decode_window_tc: out / packed must be 16-byte aligned");
        return RF_EINVAL;
    }
    Args A{};
    int rfield = 0;
    for (int i = 0; i < n_layers; ++i) {
        if (dilations[i] < 1 || dilations[i] > kPad) {
            set_error("rf_decode_window_tc: dilation %d outside [1, %d]", dilations[i], kPad);
            return RF_EINVAL;
        }
        A.dil[i] = dilations[i];
        rfield += dilations[i];
    }
    if (rfield > kMaxRF) {
        set_error("rf_decode_window_tc: receptive field %d > %d", rfield, kMaxRF);
        return RF_EINVAL;
    }
    A.latent = latent;
    A.frames = frames;
    A.C = (int)channels;
    A.packed = (const uint8_t *)packed;
    A.L = n_layers;
    A.rf = rfield;
    if (full) {
        A.vlo = 0;
        A.vhi = frames;
    } else {
        const int64_t lo = start - overlap, hi = stop + overlap;
        A.vlo = lo > 0 ? lo : 0;
        A.vhi = hi < frames ? hi : frames;
    }
    A.start = start;
    A.nout = stop - start;
    A.hop = hop;
    A.cw = g.cw;
    A.nch = g.nch;
    A.out = out;
    A.trace = g_dtrace;
    const int P = kRows - 2 * rfield;
    const int64_t tiles = (A.nout + P - 1) / P;
    // column slices: fill the SMs once (a slice recomputes its tile's conv stack)
    int64_t slices = sm_count() / tiles;
    if (slices < 1) slices = 1;
    if (slices > g.nch) slices = g.nch;
    A.slices = (int)slices;
    void (*kern)(Args) = g.CP == 16 ? rf_decode_tc_kernel<16> : g.CP == 32 ? rf_decode_tc_kernel<32>
                       : g.CP == 48 ? rf_decode_tc_kernel<48> : rf_decode_tc_kernel<64>;
    const uint32_t smem = g.CP == 16 ? Smem<16>::TOTAL : g.CP == 32 ? Smem<32>::TOTAL
                        : g.CP == 48 ? Smem<48>::TOTAL : Smem<64>::TOTAL;
    RF_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RF_TRY_CUDA(launch_pdl(kern, dim3((unsigned)(tiles * slices)), dim3(kThreads), smem, (cudaStream_t)stream, A));
    RF_TRY_LAUNCH("rf_decode_tc_kernel");
    return RF_OK;
}

// Debugging aid (not part of the product ABI): globaltimer stamps of every decode CTA
// ([cta][32] u64: phases of the conv stack / upsampler) -- see tools/decode_trace.py.
extern "C" void rf_decode_set_trace(void *buf) { rf::dtc::g_dtrace = (unsigned long long *)buf; }
