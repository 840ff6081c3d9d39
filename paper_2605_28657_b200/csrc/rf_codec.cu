// Windowed / full toy-codec decode (reference codec.py:93-164).
//
// Two kernels:
//   rf_conv_stack   : for each trimmed output frame, the dilated conv stack
//                     (kernel 3, tanh, zero outside the valid range) evaluated on a
//                     halo-staged shared-memory tile -> h[F_out, C] (float64).
//   rf_upsample_q16 : the per-frame linear upsampler h @ U^T as a register-tiled GEMM
//                     (M = output frames, N = hop, K = C) with quantize_pcm fused in
//                     the epilogue -> int16 samples.
// Every layer value at global frame g is a fixed-order sum over (tap 0,1,2) x (input
// channel 0..C-1) of values that are zero outside [vlo, vhi) -- the same in the full
// and the windowed decode -- so windowed == full holds bit for bit on the GPU whenever
// overlap >= receptive field (the reference's contract, codec.py:1-11).
#include <math.h>

#include "rf_common.cuh"

namespace rf {

constexpr int kConvThreads = 256;
constexpr int kConvTile = 16;  // output frames per CTA
constexpr int kMaxC = 64;

struct ConvArgs {
    const double *latent;
    int64_t frames, C;
    const double *kernels;  // [L,3,C,C] (tap, in k, out c)
    int32_t dil[RF_MAX_CODEC_LAYERS];
    int32_t L, rf;          // rf = sum of dilations
    int64_t vlo, vhi;       // valid global frame range
    int64_t start, nout;    // trimmed output frames [start, start+nout)
    double *h;              // [nout, C]
};

// Shared tile covers global frames [g0 - rf, g0 + kConvTile + rf).
__global__ void __launch_bounds__(kConvThreads)
rf_conv_stack(const __grid_constant__ ConvArgs A) {
    extern __shared__ double sm[];
    const int C = (int)A.C;
    const int W = kConvTile + 2 * A.rf;  // tile width in frames
    double *buf0 = sm, *buf1 = sm + (int64_t)W * C;
    const int64_t g0 = A.start + (int64_t)blockIdx.x * kConvTile;
    const int64_t gbase = g0 - A.rf;
    for (int idx = threadIdx.x; idx < W * C; idx += blockDim.x) {
        int w = idx / C, c = idx % C;
        int64_t g = gbase + w;
        buf0[idx] = (g >= A.vlo && g < A.vhi) ? A.latent[g * C + c] : 0.0;
    }
    __syncthreads();
    // layer l valid computed region shrinks by the remaining dilations
    int lo = 0, hi = W;  // region of buf holding correct values for the current layer input
    double *in = buf0, *out = buf1;
    for (int l = 0; l < A.L; ++l) {
        const int d = A.dil[l];
        const int olo = lo + d, ohi = hi - d;  // frames whose taps stay inside [lo, hi)
        const double *K = A.kernels + (int64_t)l * 3 * C * C;
        const int n = (ohi - olo) * C;
        for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
            const int w = olo + idx / C, c = idx % C;
            const int64_t g = gbase + w;
            double acc = 0.0;
            if (g >= A.vlo && g < A.vhi) {
                double tap_sum[3];
#pragma unroll
                for (int tap = 0; tap < 3; ++tap) {
                    const double *row = in + (int64_t)(w + (tap - 1) * d) * C;
                    const double *kk = K + (int64_t)tap * C * C + c;
                    double s = 0.0;
                    for (int k = 0; k < C; ++k) s = fma(row[k], kk[(int64_t)k * C], s);
                    tap_sum[tap] = s;
                }
                acc = tanh((tap_sum[0] + tap_sum[1]) + tap_sum[2]);
            }
            out[w * C + c] = acc;
        }
        __syncthreads();
        lo = olo;
        hi = ohi;
        double *t = in;
        in = out;
        out = t;
    }
    // lo..hi now equals [rf, rf + kConvTile)
    for (int idx = threadIdx.x; idx < kConvTile * C; idx += blockDim.x) {
        const int w = idx / C, c = idx % C;
        const int64_t o = (int64_t)blockIdx.x * kConvTile + w;
        if (o < A.nout) A.h[o * C + c] = in[(A.rf + w) * C + c];
    }
}

// quantize_pcm (codec.py:27-31): copysign(floor(|32767 s| + 0.5), s), clip, int16.
__device__ __forceinline__ int16_t quantize_pcm(double s) {
    double scaled = __dmul_rn(s, 32767.0);
    double r = copysign(floor(__dadd_rn(fabs(scaled), 0.5)), scaled);
    r = fmin(fmax(r, -32768.0), 32767.0);
    return (int16_t)(int)r;
}

constexpr int kUpTM = 32, kUpTN = 128, kUpThreads = 256;
// each thread: 4 frames x 4 samples

__global__ void __launch_bounds__(kUpThreads)
rf_upsample_q16(const double *__restrict__ h, const double *__restrict__ U, int64_t nout,
                int64_t hop, int C, int16_t *__restrict__ out) {
    extern __shared__ double sm[];
    double *sh = sm;                 // [kUpTM][C+1]
    double *su = sm + kUpTM * (C + 1);  // [kUpTN][C+1]
    const int64_t f0 = (int64_t)blockIdx.y * kUpTM, j0 = (int64_t)blockIdx.x * kUpTN;
    for (int idx = threadIdx.x; idx < kUpTM * C; idx += blockDim.x) {
        int r = idx / C, k = idx % C;
        sh[r * (C + 1) + k] = (f0 + r < nout) ? h[(f0 + r) * C + k] : 0.0;
    }
    for (int idx = threadIdx.x; idx < kUpTN * C; idx += blockDim.x) {
        int r = idx / C, k = idx % C;
        su[r * (C + 1) + k] = (j0 + r < hop) ? U[(j0 + r) * C + k] : 0.0;
    }
    __syncthreads();
    const int tr = threadIdx.x / 32;  // 8 row groups of 4 frames
    const int tc = threadIdx.x % 32;  // 32 column groups of 4 samples (strided by 32)
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k = 0; k < C; ++k) {
        double hv[4], uv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) hv[a] = sh[(tr * 4 + a) * (C + 1) + k];
#pragma unroll
        for (int b = 0; b < 4; ++b) uv[b] = su[(tc + 32 * b) * (C + 1) + k];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(hv[a], uv[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        int64_t f = f0 + tr * 4 + a;
        if (f >= nout) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            int64_t j = j0 + tc + 32 * b;
            if (j < hop) out[f * hop + j] = quantize_pcm(acc[a][b]);
        }
    }
}

}  // namespace rf

using namespace rf;

extern "C" int64_t rf_decode_workspace_bytes(int64_t out_frames, int64_t channels) {
    return ((out_frames * channels * 8) + 255) / 256 * 256;
}

extern "C" int rf_decode_window(const double *latent, int64_t frames, int64_t channels,
                                const double *kernels, const int32_t *dilations, int32_t n_layers,
                                const double *upsample, int64_t hop, int64_t start, int64_t stop,
                                int64_t overlap, int32_t full, int16_t *out, void *workspace,
                                int64_t workspace_bytes, void *stream) {
    if (!latent || !kernels || !dilations || !upsample || !out || !workspace) {
        set_error("rf_decode_window: null argument");
        return RF_EINVAL;
    }
    if (channels < 1 || channels > kMaxC || n_layers < 1 || n_layers > RF_MAX_CODEC_LAYERS || hop < 1) {
        set_error("rf_decode_window: unsupported shape (C=%lld, L=%d, hop=%lld)", (long long)channels,
                  n_layers, (long long)hop);
        return RF_EINVAL;
    }
    if (!(0 <= start && start < stop && stop <= frames) || overlap < 0) {
        set_error("rf_decode_window: window (%lld, %lld) outside [0, %lld)", (long long)start,
                  (long long)stop, (long long)frames);
        return RF_EINVAL;
    }
    const int64_t nout = stop - start;
    if (workspace_bytes < rf_decode_workspace_bytes(nout, channels)) {
        set_error("rf_decode_window: workspace too small");
        return RF_EWORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    ConvArgs A{};
    A.latent = latent;
    A.frames = frames;
    A.C = channels;
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
    A.nout = nout;
    A.h = (double *)workspace;
    const int W = kConvTile + 2 * rfield;
    size_t smem = (size_t)2 * W * channels * sizeof(double);
    if (smem > 200 * 1024) {
        set_error("rf_decode_window: receptive field too large for one tile");
        return RF_EINVAL;
    }
    RF_TRY_CUDA(cudaFuncSetAttribute(rf_conv_stack, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    unsigned nblk = (unsigned)((nout + kConvTile - 1) / kConvTile);
    rf_conv_stack<<<nblk, kConvThreads, smem, st>>>(A);
    RF_TRY_LAUNCH("rf_conv_stack");
    size_t smem_up = (size_t)(kUpTM + kUpTN) * (channels + 1) * sizeof(double);
    RF_TRY_CUDA(cudaFuncSetAttribute(rf_upsample_q16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_up));
    dim3 g((unsigned)((hop + kUpTN - 1) / kUpTN), (unsigned)((nout + kUpTM - 1) / kUpTM));
    rf_upsample_q16<<<g, kUpThreads, smem_up, st>>>(A.h, upsample, nout, hop, (int)channels, out);
    RF_TRY_LAUNCH("rf_upsample_q16");
    return RF_OK;
}
