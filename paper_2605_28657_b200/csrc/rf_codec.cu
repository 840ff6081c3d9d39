// Windowed / full toy-codec decode in ONE launch (reference
// codec.py:93-164).
//
// Layout: a thread-block cluster of NC (= 8) CTAs owns a tile of TF output frames.
//   * Every CTA stages the tile's input frames plus the receptive-field halo
//     [g0 - rf, g0 + TF + rf) for all C channels in shared memory (zero outside the
//     valid range [vlo, vhi), exactly the zeros the reference's padding/mask produce).
//   * Layer l: CTA r computes output channels [r*C/NC, (r+1)*C/NC) for the frames whose
//     taps stay inside the staged region (the region shrinks by d_l per side), with
//     its slice of the conv weights resident in shared memory.  Each output is a
//     fixed-order sum (8 lanes x C/8 input channels x 3 taps, fixed shuffle tree), tanh,
//     and zero outside [vlo, vhi).  A group of 8 lanes computes all of the CTA's C/NC
//     channels of one frame: every activation load feeds C/NC independent FMA chains, the
//     weights are stored [tap][k/8][channel][k%8] so the 8 lanes read consecutive doubles,
//     activation rows are padded by 8 doubles (two groups' rows fall on different banks),
//     and after the reduction tree lane j applies tanh to channel j.
//   * After each layer the cluster synchronises and every CTA gathers the other CTAs'
//     channel slices through distributed shared memory (DSMEM), so activations never
//     leave the SMs.
//   * Finally CTA r computes samples [r*hop/NC, (r+1)*hop/NC) of every tile frame:
//     pcm[f][j] = quantize(sum_c h[f][c] * U[j][c]), with U^T streamed from L2 and the
//     int16 rounding/clipping of quantize_pcm (codec.py:27-31) fused.
// Because every value at global frame g is computed by the same fixed-order arithmetic
// whatever the window, windowed == full holds bit for bit on the GPU whenever
// overlap >= receptive field (the reference's contract, codec.py:1-11).
#include <cooperative_groups.h>
#include <math.h>

#include "rf_common.cuh"

namespace cg = cooperative_groups;

namespace rf {

constexpr int kNC = 8;          // CTAs per cluster
// output frames per cluster: 16, or 8 for short windows (twice the clusters: a 3-s window
// then spreads over 80 instead of 40 SMs; per-frame arithmetic is independent of the tiling)
constexpr int kThreads = 256;
constexpr int kKS = 8;          // lanes cooperating on one conv output
constexpr int kMaxC = 64;

struct DecodeArgs {
    const double *latent;       // [frames, C]
    int64_t frames;
    int C, CS;                  // channels, channels per CTA (informational)
    const double *kernels;      // [L,3,C,C] (tap, in k, out c)
    int32_t dil[RF_MAX_CODEC_LAYERS];
    int32_t L, rf;
    int64_t vlo, vhi;           // valid global frame range
    int64_t start, nout;        // output frames [start, start + nout)
    const double *upT;          // [C, hop] (transposed upsampler)
    int64_t hop;
    int16_t *out;               // [nout * hop]
};

// quantize_pcm (codec.py:27-31): copysign(floor(|32767 s| + 0.5), s), clip, int16.
__device__ __forceinline__ int16_t quantize_pcm(double s) {
    double scaled = __dmul_rn(s, 32767.0);
    double r = copysign(floor(__dadd_rn(fabs(scaled), 0.5)), scaled);
    r = fmin(fmax(r, -32768.0), 32767.0);
    return (int16_t)(int)r;
}

template <int C, int kTF>
__global__ void __launch_bounds__(kThreads)
rf_decode_cluster(const __grid_constant__ DecodeArgs A) {
    constexpr int CS = C / kNC;       // output channels per CTA
    constexpr int KPER = C / kKS;     // input channels per lane of a conv output
    constexpr int ACS = C + 8;        // padded activation row (bank spread across frame rows)
    extern __shared__ __align__(16) double sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int L = A.L;
    const int W = kTF + 2 * A.rf;
    const int jper = (int)((A.hop + kNC - 1) / kNC);
    double *act = sm;                                   // [W][ACS] current layer input
    double *part0 = act + (size_t)W * ACS;              // [2][W][CS] this CTA's layer output
    double *wts = part0 + (size_t)2 * W * CS;           // [L][3][C/8][CS][8] (tap, k/8, out, k%8)
    double *hT = wts + (size_t)L * 3 * C * CS;          // [C][kTF] final layer, transposed
    double *ups = hT + (size_t)C * kTF;                 // [C][jper] this CTA's U^T slice
    const int c0 = rank * CS;
    // persistent clusters: cluster q decodes tiles q, q + nclusters, ...; the weight and
    // upsampler slices are staged once per CTA, the latent tile + halo once per tile
    const int64_t ntiles = (A.nout + kTF - 1) / kTF;
    const int64_t nclusters = gridDim.x / kNC;

    // the tile + halo (16-byte cp.async granules, zero-fill outside the valid frame range)
    auto stage_tile = [&](int64_t gbase) {
        constexpr int C2 = C / 2;
        for (int w = threadIdx.x / C2; w < W; w += kThreads / C2) {
            const int c = 2 * (threadIdx.x % C2);
            const int64_t g = gbase + w;
            const bool in = g >= A.vlo && g < A.vhi;
            const unsigned dst = (unsigned)__cvta_generic_to_shared(act + w * ACS + c);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst),
                         "l"(A.latent + (in ? g * C + c : 0)), "r"(in ? 16 : 0));
        }
    };
    // Groups: weights + the first tile, then this CTA's upsampler slice, which the first
    // tile only waits for after its conv layers.
    for (int rest = threadIdx.x / CS; rest < L * 3 * C; rest += kThreads / CS) {
        const int cc = threadIdx.x % CS;                // rest = (l*3 + tap)*C + k
        const int lt = rest / C, k = rest % C;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(
            wts + (((size_t)lt * KPER + k / kKS) * CS + cc) * kKS + k % kKS);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                     "l"(A.kernels + (int64_t)rest * C + c0 + cc));
    }
    if (blockIdx.x / kNC < ntiles) stage_tile(A.start + (blockIdx.x / kNC) * kTF - A.rf);
    asm volatile("cp.async.commit_group;\n" ::);
    const int j0 = rank * jper;
    const int jn = (int)(j0 + jper < A.hop ? jper : A.hop - j0);
    // U^T slice: 16-byte granules when both row starts are 16-byte aligned (hop, jper even)
    const bool up16 = ((A.hop | jper | j0) & 1) == 0;
    const int jq = up16 ? (jn + 1) / 2 : jn;   // granules per row
    for (int e = threadIdx.x; e < C * jq; e += kThreads) {
        const int c = e / jq, q = e % jq;
        const double *src = A.upT + (int64_t)c * A.hop + j0;
        if (up16 && 2 * q + 1 < jn) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(ups + (size_t)c * jper + 2 * q);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + 2 * q));
        } else {
            const int jj = up16 ? 2 * q : q;
            const unsigned dst = (unsigned)__cvta_generic_to_shared(ups + (size_t)c * jper + jj);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src + jj));
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  bool first = true;
  for (int64_t tile = blockIdx.x / kNC; tile < ntiles; tile += nclusters) {
    const int64_t g0 = A.start + tile * kTF;
    const int64_t gbase = g0 - A.rf;
    if (!first) {
        stage_tile(gbase);
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_all;\n" ::);
    } else {
        asm volatile("cp.async.wait_group 1;\n" ::);   // weights + first tile; U^T may still fly
    }
    __syncthreads();

    const int grp = threadIdx.x / kKS, sub = threadIdx.x % kKS;
    constexpr int ngrp = kThreads / kKS;
    int lo = 0, hi = W;
    for (int l = 0; l < L; ++l) {
        const int d = A.dil[l];
        const int olo = lo + d, ohi = hi - d;
        const double *K = wts + (size_t)l * 3 * C * CS;
        const int nf = ohi - olo;                             // frames of this layer
        double *part = part0 + (size_t)(l & 1) * W * CS;  // double-buffered across layers
        for (int base = 0; base < nf; base += ngrp) {
            const int fi = base + grp;
            const bool live = fi < nf;
            const int w = live ? olo + fi : olo;
            double s0[CS], s1[CS], s2[CS];
#pragma unroll
            for (int cc = 0; cc < CS; ++cc) s0[cc] = s1[cc] = s2[cc] = 0.0;
            if (live) {
                // lane `sub` takes input channels sub, sub+8, ...: the 8 lanes of a group
                // read consecutive doubles of the activations and of the weights
                const double *r0 = act + (w - d) * ACS + sub;
                const double *r1 = act + w * ACS + sub;
                const double *r2 = act + (w + d) * ACS + sub;
                const double *kk = K + sub;
#pragma unroll
                for (int k = 0; k < KPER; ++k) {
                    const double a0 = r0[k * kKS], a1 = r1[k * kKS], a2 = r2[k * kKS];
                    const double *k0 = kk + ((0 * KPER + k) * CS) * kKS;
                    const double *k1 = kk + ((1 * KPER + k) * CS) * kKS;
                    const double *k2 = kk + ((2 * KPER + k) * CS) * kKS;
#pragma unroll
                    for (int cc = 0; cc < CS; ++cc) {
                        s0[cc] = fma(a0, k0[cc * kKS], s0[cc]);
                        s1[cc] = fma(a1, k1[cc * kKS], s1[cc]);
                        s2[cc] = fma(a2, k2[cc * kKS], s2[cc]);
                    }
                }
            }
            double mine = 0.0;
#pragma unroll
            for (int cc = 0; cc < CS; ++cc) {
                double s = __dadd_rn(__dadd_rn(s0[cc], s1[cc]), s2[cc]);
                // fixed 8-lane reduction tree (the lanes of a group are adjacent)
                s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
                s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
                s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
                if (cc == sub % CS) mine = s;
            }
            if (live && sub < CS) {   // lane j: channel j (tanh spread over the group)
                const int64_t g = gbase + w;
                part[w * CS + sub] = (g >= A.vlo && g < A.vhi) ? tanh(mine) : 0.0;
            }
        }
        cluster.sync();   // every CTA's slice of layer l is complete (and, because each
                          // CTA computed layer l after gathering layer l-1, nobody still
                          // reads the other `part` buffer, which layer l+1 overwrites)
        // gather all slices of rows [olo, ohi) through DSMEM, 4 remote loads in flight
        const bool last = l == L - 1;
        constexpr int RPI = kThreads / C;             // rows per pass
        const int c = threadIdx.x % C;
        const double *rp = cluster.map_shared_rank(part, c / CS);
        for (int w0 = olo + threadIdx.x / C; w0 < ohi; w0 += 4 * RPI) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int w = w0 + u * RPI;
                v[u] = w < ohi ? rp[w * CS + c % CS] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int w = w0 + u * RPI;
                if (w < ohi) {
                    if (last)
                        hT[c * kTF + (w - olo)] = v[u];
                    else
                        act[w * ACS + c] = v[u];
                }
            }
        }
        __syncthreads();  // this CTA's act is complete before computing the next layer
        lo = olo;
        hi = ohi;
    }
    cluster.sync();   // no CTA may exit (or restage) while a peer could still read its `part`
    if (first) {
        asm volatile("cp.async.wait_all;\n" ::);   // the upsampler slice
        __syncthreads();
        first = false;
    }
    // pcm[f][j] = quantize(sum_c h[f][c] U[j][c]) for this CTA's samples
    const int64_t fmax = A.nout - tile * kTF < kTF ? A.nout - tile * kTF : kTF;
    for (int jj = threadIdx.x; jj < jn; jj += kThreads) {
        double acc[kTF];
#pragma unroll
        for (int f = 0; f < kTF; ++f) acc[f] = 0.0;
#pragma unroll 4
        for (int c = 0; c < C; ++c) {
            const double u = ups[c * jper + jj];
            const double2 *hv = reinterpret_cast<const double2 *>(hT + c * kTF);
#pragma unroll
            for (int f2 = 0; f2 < kTF / 2; ++f2) {
                const double2 h = hv[f2];
                acc[2 * f2] = fma(h.x, u, acc[2 * f2]);
                acc[2 * f2 + 1] = fma(h.y, u, acc[2 * f2 + 1]);
            }
        }
        const int64_t j = j0 + jj;
#pragma unroll
        for (int f = 0; f < kTF; ++f)
            if (f < fmax) A.out[(tile * kTF + f) * A.hop + j] = quantize_pcm(acc[f]);
    }
    __syncthreads();   // hT and act are read before the next tile overwrites them
  }
}

}  // namespace rf

using namespace rf;

extern "C" int64_t rf_decode_workspace_bytes(int64_t out_frames, int64_t channels) {
    (void)out_frames;
    (void)channels;
    return 256;  // the fused kernel keeps every intermediate on chip
}

extern "C" int rf_decode_window(const double *latent, int64_t frames, int64_t channels,
                                const double *kernels, const int32_t *dilations, int32_t n_layers,
                                const double *upsample_t, int64_t hop, int64_t start, int64_t stop,
                                int64_t overlap, int32_t full, int16_t *out, void *workspace,
                                int64_t workspace_bytes, void *stream) {
    (void)workspace;
    (void)workspace_bytes;
    if (!latent || !kernels || !dilations || !upsample_t || !out) {
        set_error("rf_decode_window: null argument");
        return RF_EINVAL;
    }
    const bool pow2 = channels >= kNC && (channels & (channels - 1)) == 0;
    if (channels < 1 || channels > kMaxC || !pow2 || n_layers < 1 ||
        n_layers > RF_MAX_CODEC_LAYERS || hop < 1) {
        set_error("rf_decode_window: unsupported shape (C=%lld must be a power of two in [%d, %d], L=%d, hop=%lld)",
                  (long long)channels, kNC, kMaxC, n_layers, (long long)hop);
        return RF_EINVAL;
    }
    if (!(0 <= start && start < stop && stop <= frames) || overlap < 0) {
        set_error("rf_decode_window: window (%lld, %lld) outside [0, %lld)", (long long)start,
                  (long long)stop, (long long)frames);
        return RF_EINVAL;
    }
    DecodeArgs A{};
    A.latent = latent;
    A.frames = frames;
    A.C = (int)channels;
    A.CS = (int)channels / kNC;
    A.kernels = kernels;
    A.L = n_layers;
    int rfield = 0;
    for (int i = 0; i < n_layers; ++i) {
        if (dilations[i] < 1) {
            set_error("rf_decode_window: dilation must be >= 1");
            return RF_EINVAL;
        }
        A.dil[i] = dilations[i];
        rfield += dilations[i];
    }
    A.rf = rfield;
    if (full) {
        A.vlo = 0;
        A.vhi = frames;
    } else {
        int64_t lo = start - overlap, hi = stop + overlap;
        A.vlo = lo > 0 ? lo : 0;
        A.vhi = hi < frames ? hi : frames;
    }
    A.start = start;
    A.nout = stop - start;
    A.upT = upsample_t;
    A.hop = hop;
    A.out = out;
    // short outputs: 8-frame tiles (more clusters in flight); long ones: 16 (less halo work)
    const int kTF = (stop - start) <= 8 * 148 / kNC * 2 ? 8 : 16;
    const int W = kTF + 2 * rfield;
    const int64_t jper = (hop + kNC - 1) / kNC;
    size_t smem = ((size_t)W * (channels + 8) + (size_t)2 * W * A.CS + (size_t)n_layers * 3 * channels * A.CS +
                   (size_t)channels * kTF + (size_t)channels * jper) * sizeof(double);
    if (smem > 220 * 1024) {
        set_error("rf_decode_window: receptive field / hop too large for one tile (%zu B smem)", smem);
        return RF_EINVAL;
    }
    void (*kern)(DecodeArgs);
    if (kTF == 8)
        kern = channels == 8 ? rf_decode_cluster<8, 8> : channels == 16 ? rf_decode_cluster<16, 8>
             : channels == 32 ? rf_decode_cluster<32, 8> : rf_decode_cluster<64, 8>;
    else
        kern = channels == 8 ? rf_decode_cluster<8, 16> : channels == 16 ? rf_decode_cluster<16, 16>
             : channels == 32 ? rf_decode_cluster<32, 16> : rf_decode_cluster<64, 16>;
    RF_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t tiles = (A.nout + kTF - 1) / kTF;
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kNC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent: as many clusters as can be co-resident (8-CTA clusters must fit in one
    // GPC, so this is below sm_count / 8); a non-resident cluster would run its whole tile
    // list after the others
    int active = 0;
    cfg.gridDim = dim3((unsigned)kNC);
    if (cudaOccupancyMaxActiveClusters(&active, (void *)kern, &cfg) != cudaSuccess || active < 1) {
        cudaGetLastError();
        active = 1;
    }
    const int64_t clusters = tiles < active ? tiles : active;
    cfg.gridDim = dim3((unsigned)(clusters * kNC));
    RF_TRY_CUDA(cudaLaunchKernelEx(&cfg, kern, A));
    return RF_OK;
}

// ------------------------------------------------------------------ encode (B-enc) ----
// ToyCodec.encode (codec.py:168-174): latent[f, c] = sum_k samples[f * hop + k] * proj[c, k],
// float64.  One CTA per frame: the frame's hop samples are staged in shared memory, thread c
// accumulates channel c over k in ascending order with FMA (fixed order, so deterministic;
// numpy's BLAS order differs, agreement to ~1e-15 relative).  proj_t is [hop, C] so the C
// threads read consecutive doubles for each k.  Off the tick (source preparation), 2 C hop
// FLOP per frame.
namespace rf {
__global__ void __launch_bounds__(128)
rf_encode_kernel(const double *__restrict__ samples, int64_t hop, const double *__restrict__ proj_t, int channels,
                 double *__restrict__ out) {
    extern __shared__ double s_frame[];
    const int64_t f = blockIdx.x;
    for (int64_t k = threadIdx.x; k < hop; k += blockDim.x) s_frame[k] = samples[f * hop + k];
    __syncthreads();
    for (int c = threadIdx.x; c < channels; c += blockDim.x) {
        double acc = 0.0;
        for (int64_t k = 0; k < hop; ++k) acc = fma(s_frame[k], proj_t[k * channels + c], acc);
        out[f * channels + c] = acc;
    }
}
}  // namespace rf

extern "C" int rf_encode_frames(const double *samples, int64_t frames, int64_t hop, const double *proj_t,
                                int64_t channels, double *latent, void *stream) {
    if (!samples || !proj_t || !latent || frames < 1 || hop < 1 || channels < 1 || channels > 1024) {
        set_error("rf_encode_frames: bad arguments (frames=%lld hop=%lld C=%lld)", (long long)frames,
                  (long long)hop, (long long)channels);
        return RF_EINVAL;
    }
    const size_t smem = (size_t)hop * sizeof(double);
    if (smem > 48 * 1024) {
        static bool attr = false;
        if (!attr) {
            RF_TRY_CUDA(cudaFuncSetAttribute(rf_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            attr = true;
        }
        if (smem > 200 * 1024) {
            set_error("rf_encode_frames: hop %lld too large", (long long)hop);
            return RF_EINVAL;
        }
    }
    rf_encode_kernel<<<(unsigned)frames, 128, smem, (cudaStream_t)stream>>>(samples, hop, proj_t, (int)channels,
                                                                             latent);
    RF_TRY_LAUNCH("rf_encode_kernel");
    return RF_OK;
}
