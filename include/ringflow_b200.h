/*
 * ringflow_b200.h -- C ABI of the B200-native per-tick streaming-diffusion hot path.
 *
 * The reference (arxiv/paper_2605_28657, package `ringflow`) is pure Python + numpy and
 * has no FFI of its own.  Each entry point below replaces the numpy
 * arithmetic behind one reference function; the Python mirror in
 * paper_2605_28657_b200/ keeps the reference's public API (StreamPipeline, ToyCodec,
 * sde_step, ...) and calls these through ctypes.  The reference-side binding a
 * maintainer would add is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Device pointers only (caller-owned, e.g. torch tensors); nothing is allocated
 *     here except where an explicit workspace argument says so.
 *   - Latents are [T, D] frame-major, C-contiguous float64 (the reference's layout,
 *     latents.py:3-6); per-frame curves are float64 [T].
 *   - Every call is asynchronous on the given stream (cudaStream_t passed as void*).
 *   - Return 0 on success or an RF_E* code; rf_last_error() describes the failure.
 */
#ifndef RINGFLOW_B200_H
#define RINGFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RF_ABI_VERSION 1

#define RF_OK 0
#define RF_EINVAL 1     /* bad argument (shape, null pointer, range) */
#define RF_ECUDA 2      /* a CUDA runtime error */
#define RF_EWORKSPACE 3 /* workspace too small */

/* Device status word bits (written by kernels, read back by the host at sync points). */
#define RF_STATUS_NOISE_SHORT 0x1u    /* a normal draw ran out of generated stream positions */
#define RF_STATUS_NOISE_LONG 0x2u     /* a single draw consumed > RF_ZIG_MAX_LEN words (slow path used) */
#define RF_STATUS_NONFINITE 0x4u      /* an emitted latent held a non-finite value */

int rf_abi_version(void);
const char *rf_last_error(void);
/* Number of SMs of the current device (grid sizing). */
int rf_device_sm_count(void);

/* ---------------------------------------------------------------- noise (A14) ----
 * Replaces NoiseSource.normal / NoiseSource.uniform (reference latents.py:117-150):
 * np.random.Generator(np.random.Philox(key)).standard_normal(n) / .random(n), bit-exact.
 * The 128-bit Philox key is the blake2b digest computed on the host
 * (latents.py:130-135); k0 = low 64 bits, k1 = high 64 bits.
 */
typedef struct rf_draw {
    uint64_t k0, k1; /* Philox4x64-10 key words */
    int64_t n;       /* number of outputs */
    double *out;     /* device [n] */
} rf_draw;

/* Workspace bytes needed to run `count` normal draws of the given sizes in one batch. */
int64_t rf_normal_workspace_bytes(const rf_draw *draws, int count);
/* Batched standard-normal fill; `draws` is a HOST array; `status` a device uint32 (OR-ed). */
int rf_normal_fill(const rf_draw *draws, int count, void *workspace, int64_t workspace_bytes,
                   uint32_t *status, void *stream);
/* Batched uniform [0,1) fill (Generator.random). */
int rf_uniform_fill(const rf_draw *draws, int count, void *stream);

/* ------------------------------------------------------ fused tick solve (A5-A12) ----
 * One launch advances every active ring row by one solver step:
 *   velocity (ToyFlowModel.velocity, model.py:133-152, one per condition)
 *   -> blend_conditions (solver.py:204-227)
 *   -> guided_velocity (solver.py:141-201; CFG / RCFG modes / APG momentum / rescale)
 *   -> sde_step (solver.py:273-306, incl. _morph_target 230-238) or ode_step (241-270).
 * Arithmetic is float64 in the reference's operation order without FMA contraction,
 * so results are bit-identical to the numpy reference given identical inputs.
 */
#define RF_MAX_COND 4
#define RF_CURVE_SDE 0        /* sde_denoise_curve  (mult) */
#define RF_CURVE_GUIDANCE 1   /* guidance_curve     (mult) */
#define RF_CURVE_VSCALE 2     /* velocity_scale     (mult) */
#define RF_CURVE_ODE_NOISE 3  /* ode_noise_curve    (add)  */
#define RF_CURVE_APG 4        /* apg_momentum       (add)  */
#define RF_CURVE_RESCALE 5    /* cfg_rescale_curve  (mult) */
#define RF_CURVE_X0_STRENGTH 6/* x0_target_strength (mult) */
#define RF_NUM_CURVES 7

#define RF_SOLVER_SDE 0
#define RF_SOLVER_ODE 1

/* Negative-velocity source for guidance this step (resolved on the host from rcfg_mode
 * and the slot's StepState, pipeline.py:436-446 / solver.py:161-180). */
#define RF_NEG_NONE 0          /* guidance disabled */
#define RF_NEG_UNCOND 1        /* off / full-cfg, or first step of the rcfg variants */
#define RF_NEG_RESIDUAL 2      /* onetime-negative: v_c - residual (residual cached) */
#define RF_NEG_PREV 3          /* self-negative: previous step's positive velocity */

typedef struct rf_row {
    double *x;                        /* [T*D] ring state, updated in place */
    const double *noise_model;        /* [T*D] n_model(step) or NULL when jitter == 0 */
    const double *noise_step;         /* [T*D] n_sde(step) / n_ode(step) or NULL */
    const double *source;             /* [T*D] or NULL */
    const double *x0_target;          /* [T*D] or NULL (morph inactive this step) */
    const double *curves[RF_NUM_CURVES]; /* [T] each or NULL (= sentinel / absent) */
    const double *cond_x0[RF_MAX_COND];  /* x0 before style offset, per condition */
    const double *cond_w[RF_MAX_COND];   /* per-frame blend weights or NULL (ones) */
    const double *uncond_x0;          /* x0 of the unconditional branch (guidance) */
    double *momentum;                 /* [T*D] APG state or NULL */
    double *residual;                 /* [T*D] onetime-negative residual or NULL */
    double *prev_positive;            /* [T*D] self-negative state or NULL */
    double *v_out;                    /* [T*D] optional copy of the final (guided) velocity */
    double t_curr, t_next;
    double jitter_t;                  /* model_jitter * t_curr (host double, model.py:151) */
    int32_t n_cond;
    int32_t solver;                   /* RF_SOLVER_* */
    int32_t neg_kind;                 /* RF_NEG_* */
    int32_t flags;                    /* RF_ROWF_* */
} rf_row;

#define RF_ROWF_MOMENTUM_INIT 0x1  /* momentum is None: start from zeros */
#define RF_ROWF_WRITE_RESIDUAL 0x2 /* onetime-negative step 0: residual = v_c - v_u */
#define RF_ROWF_WRITE_PREV 0x4     /* self-negative: store prev_positive = v_c */
#define RF_ROWF_ODE_MORPH 0x8      /* ODE with an active x0 target (solver.py:261-263) */
#define RF_ROWF_COND_V 0x10        /* cond_x0[k] hold velocities (DiT output / seam input) */
#define RF_ROWF_UNCOND_V 0x20      /* uncond_x0 holds the negative velocity */
#define RF_ROWF_NO_STEP 0x40       /* velocity only (guided_velocity seam): x untouched */
#define RF_ROWF_V_F32 0x80         /* cond/uncond velocities are float32 (DiT output) */
#define RF_ROWF_STYLE_V 0x100      /* given velocities get the shared style offset applied in
                                      x0 space: v' = v - style/t_curr (model.py:123-131's
                                      x0 + style_offset for a velocity-predicting model) */

/* rows: HOST array of `count` rows; style_offset: device [T*D] (ModelWeights). */
int rf_tick_solve(const rf_row *rows, int count, int64_t frames, int64_t channels,
                  const double *style_offset, void *stream);

/* -------------------------------------------------------- admission (A17) --------
 * _admit (pipeline.py:523-542): x = noise if denoise == 1 else d*noise + (1-d)*source. */
typedef struct rf_admit {
    double *x;
    const double *noise;
    const double *source; /* NULL when denoise == 1 */
    double denoise;
} rf_admit;
int rf_admit_init(const rf_admit *admits, int count, int64_t numel, void *stream);

/* x0_of (model.py:123-131): out = ((base [+ hs*hint]) [+ ts*timbre]) [+ style], a term
 * being skipped when its pointer is NULL; hs/ts are the host-side products
 * strength * 0.45.  Same operation order as the reference. */
int rf_x0_compose(double *out, const double *base, const double *hint, double hs,
                  const double *timbre, double ts, const double *style, int64_t numel,
                  void *stream);

/* ------------------------------------------------------------ emit (A16) ---------
 * _emit (pipeline.py:466-491): for each emitted latent e (in emit order), copy it to
 * its record buffer, flag non-finite values, and compute
 *   mse_prev[e] = mean((lat_e - prev_e)^2), prev_e = lat_{e-1} (or `last` for e = 0)
 *   mse_ref[e]  = mean((lat_e - reference)^2)
 * with a fixed-order (deterministic) reduction.  `prev`/`reference` may be NULL.
 * Any count: emits run in launches of 16, each chunk's first prev being the previous
 * chunk's last latent.  scratch: device doubles owned by the caller (one buffer per
 * stream), at least rf_reduce_workspace_elems(numel), ZEROED before its first use: its
 * tail holds per-emit completion counters, which every call leaves zero again. */
typedef struct rf_emit {
    const double *latent; /* slot state */
    double *record;       /* record-owned copy */
} rf_emit;
int rf_emit_stats(const rf_emit *emits, int count, int64_t numel, const double *last,
                  const double *reference, double *mse_prev, double *mse_ref,
                  uint32_t *status, double *scratch, int64_t scratch_elems, void *stream);
/* Scratch doubles rf_emit_stats / rf_mse need for latents of `numel` elements. */
int64_t rf_reduce_workspace_elems(int64_t numel);

/* ------------------------------------------------------------- codec (B1-B9) -----
 * ToyCodec (codec.py:67-174).  The decode of an extended window [F, C] runs the
 * dilated conv stack (tanh, valid-row mask), the per-frame upsampler and
 * quantize_pcm in one clustered kernel, writing only the trimmed samples.
 *   latent: device [frames, C]; kernels: device [L, 3, C, C];
 *   upsample_t: device [C, hop] (the reference's [hop, C] upsampler, transposed);
 *   C must be a multiple of 8 and <= 64.
 *   window [start, stop) and overlap as in windowed_decode (codec.py:136-164);
 *   full_decode is the window [0, frames) with overlap 0 and no mask.
 *   out: device int16 [(stop - start) * hop].
 *   dilations: HOST array of n_layers (<= RF_MAX_CODEC_LAYERS).
 *   workspace: device, >= rf_decode_workspace_bytes(stop - start, channels). */
#define RF_MAX_CODEC_LAYERS 8
int64_t rf_decode_workspace_bytes(int64_t out_frames, int64_t channels);
int rf_decode_window(const double *latent, int64_t frames, int64_t channels,
                     const double *kernels, const int32_t *dilations, int32_t n_layers,
                     const double *upsample_t, int64_t hop, int64_t start, int64_t stop,
                     int64_t overlap, int32_t full, int16_t *out, void *workspace,
                     int64_t workspace_bytes, void *stream);

/* The same decode on the tensor cores (csrc/rf_decode_tc.cu): the conv stack and the
 * upsampler as implicit GEMMs (tcgen05 kind::f16, every operand split into two fp16
 * pieces hi + lo, three MMAs per product, fp32 accumulation), quantize_pcm fused; within
 * 1 LSB of the float64 reference, windowed == full bit for bit when overlap >= rf.
 * Shapes: C <= 64, hop a multiple of 16, dilations <= 16, receptive field <= 56; anything
 * else uses rf_decode_window.  rf_decode_tc_packed_bytes returns 0 for an unsupported
 * shape.  rf_decode_tc_pack converts the float64 weights once (codec construction) into
 * `packed` (device, 16-byte aligned); rf_decode_window_tc then reads only `packed`.
 *   out: device int16 [(stop - start) * hop], 16-byte aligned. */
int64_t rf_decode_tc_packed_bytes(int64_t channels, int64_t hop, int32_t n_layers);
int rf_decode_tc_pack(const double *kernels, int32_t n_layers, int64_t channels,
                      const double *upsample_t, int64_t hop, void *packed, int64_t packed_bytes,
                      void *stream);
int rf_decode_window_tc(const double *latent, int64_t frames, int64_t channels, const void *packed,
                        const int32_t *dilations, int32_t n_layers, int64_t hop, int64_t start,
                        int64_t stop, int64_t overlap, int32_t full, int16_t *out, void *stream);

/* ToyCodec.encode (codec.py:168-174): latent[f, c] = sum_k samples[f*hop + k] * proj[c, k].
 *   samples: device float64 [frames * hop]; proj_t: device [hop, C] (the reference's
 *   encode_proj [C, hop], transposed); latent: device float64 [frames, C]. */
int rf_encode_frames(const double *samples, int64_t frames, int64_t hop, const double *proj_t,
                     int64_t channels, double *latent, void *stream);

/* ------------------------------------------------------------ DiT GEMM (A8) ------
 * The tensor-core GEMM of the ACE-Step-shape DiT velocity model (the reference's
 * ToyFlowModel slot, model.py:91-152): out[M,N] = A[M,K] * B[N,K]^T with bf16 operands
 * (both K-major, nn.Linear layout), fp32 accumulation in TMEM (tcgen05.mma fed by TMA).
 * epilogue: 0 = store bf16, 1 = store f32, 2 = f32 gated residual
 *   out[m,n] += gate[(m / rows_per_batch) * gate_ld + n] * acc, 3 = SwiGLU over
 *   interleaved (gate, up) columns -> bf16 out[m, n/2], 4 = store f32 * alpha.
 * K % 64 == 0, N % block_n == 0, block_n in {128, 256}: one CTA per 128 x block_n tile;
 * -block_n: a CTA pair (cta_group::2) per 256 x block_n tile; |block_n| + 4096: stream-K
 * tile walk (equal k-block shares per persistent CTA; split tiles summed in a fixed order). */
#define RF_EPI_BF16 0
#define RF_EPI_F32 1
#define RF_EPI_RESID_GATE 2
#define RF_EPI_SWIGLU 3
#define RF_EPI_F32_SCALE 4
int rf_gemm_bf16(const void *A, const void *B, void *out, int64_t M, int64_t N, int64_t K, int64_t lda,
                 int64_t ldb, int64_t ldo, int32_t epilogue, const float *gate, int64_t gate_ld,
                 int32_t rows_per_batch, float alpha, int32_t block_n, void *stream);

/* Multi-head attention on tcgen05/TMEM (single-pass online softmax, bf16 in/out, fp32
 * softmax and accumulation), head_dim 128: q [batch*n_q, ldq] (head h at column h*128),
 * k [batch*n_k, ldk] with kv head h / (heads / kv_heads); V is given transposed:
 * vt [batch, kv_heads, 128, n_k_pad] (keys contiguous, pad columns zero);
 * out [batch*n_q, ldo]. */
int rf_attention_tc_bf16(const void *q, const void *k, const void *vt, void *out, int32_t batch, int32_t n_q,
                         int32_t n_k, int32_t n_k_pad, int32_t heads, int32_t kv_heads, int64_t ldq, int64_t ldk,
                         int64_t ldo, void *stream);
/* The same with the kernel for > 128 keys chosen explicitly (benchmarks / tests; the DiT
 * forward always uses kernel 0, the default): 0 = default, 1 = 64-key tiles with
 * double-buffered scores, one head per CTA (non-persistent). */
int rf_attention_tc_bf16_kernel(int32_t kernel, const void *q, const void *k, const void *vt, void *out,
                                int32_t batch, int32_t n_q, int32_t n_k, int32_t n_k_pad, int32_t heads,
                                int32_t kv_heads, int64_t ldq, int64_t ldk, int64_t ldo, void *stream);

/* --------------------------------------------------- ACE-Step-shape DiT (A8) ------
 * The velocity model that replaces the reference's ToyFlowModel for BASELINE configs
 * 2-5 (the reference has no DiT: builder-defined ACE-Step-1.5 shape).
 * rows = ring slots x conditions (+ unconditional rows for guidance), each with its
 * own timestep t (its schedule's sigma[step]) and conditioning tokens. */
typedef struct rf_dit_config {
    int32_t latent_channels; /* 64 */
    int32_t patch;           /* 2: tokens = frames / 2 */
    int32_t d_model;         /* 2048 */
    int32_t n_layers;        /* 24 */
    int32_t n_heads;         /* 16 */
    int32_t n_kv_heads;      /* 8 (GQA) */
    int32_t head_dim;        /* 128 */
    int32_t mlp_hidden;      /* 6144 (SwiGLU) */
    int32_t n_cond_tokens;   /* 128 */
    int32_t freq_dim;        /* 256 (sinusoidal timestep features) */
    float rope_theta;        /* 10000 */
    float norm_eps;          /* 1e-6 */
} rf_dit_config;

typedef struct rf_dit_weights { /* device pointers, bf16 [out, in] unless noted */
    const void *w_in;        /* [d, patch*C] */
    const void *w_t1;        /* [d, freq_dim] */
    const void *w_t2;        /* [d, d] */
    const void *w_ada;       /* [6d, d]   AdaLN-single */
    const float *ada_table;  /* [L, 6d] f32 per-layer modulation table */
    const void *w_qkv;       /* [L][(H + 2 Hkv) * 128, d] */
    const void *w_o;         /* [L][d, H * 128] */
    const void *w_qc;        /* [L][H * 128, d] */
    const void *w_kvc;       /* [L][2 Hkv * 128, d] */
    const void *w_oc;        /* [L][d, H * 128] */
    const void *w_gu;        /* [L][2 F, d] rows interleaved (gate_j, up_j) */
    const void *w_down;      /* [L][d, F] */
    const void *w_final_ada; /* [2d, d] */
    const void *w_out;       /* [patch*C, d] */
    const float *ones;       /* [d] f32 ones (ungated residual) */
} rf_dit_weights;

int64_t rf_dit_workspace_bytes(const rf_dit_config *cfg, int32_t max_rows, int32_t frames);
int rf_dit_create(const rf_dit_config *cfg, const rf_dit_weights *w, int32_t max_rows, int32_t frames,
                  void *workspace, int64_t workspace_bytes, void **handle, void *stream);
int rf_dit_destroy(void *handle);
/* x_rows/cond_rows: HOST arrays of device pointers (float64 [frames*C] latents,
 * bf16 [n_cond_tokens, d] conditioning); t_rows: HOST float timesteps.  v_out: device
 * f32 [rows, frames*C] or NULL for the handle's own buffer (rf_dit_output). */
int rf_dit_forward(void *handle, int32_t rows, const double *const *x_rows, const float *t_rows,
                   const void *const *cond_rows, float *v_out, void *stream);
float *rf_dit_output(void *handle);

/* Squared-difference reduction used by the similarity filter and tests (fixed order). */
int rf_mse(const double *a, const double *b, int64_t numel, double *out, double *scratch,
           int64_t scratch_elems, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* RINGFLOW_B200_H */
