// Fused per-tick solver: toy velocity + condition blend + guidance + SDE/ODE update
// for every active ring row in one launch.
//
// Reference semantics, in the reference's floating-point operation order:
//   ToyFlowModel.velocity     model.py:133-152   v = (x - x0)/t + (jitter*t)*n_model
//   x0_of                     model.py:123-131   x0 = partial(prompt,hint,timbre) + style_offset
//   blend_conditions          solver.py:204-227  v = (sum w_i v_i) / (sum w_i)
//   guided_velocity           solver.py:141-201  CFG / RCFG / APG momentum / rescale
//   _morph_target             solver.py:230-238
//   sde_step                  solver.py:273-306
//   ode_step                  solver.py:241-270
// Every floating-point operation uses an explicit round-to-nearest intrinsic
// (__dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn) so nvcc cannot contract to FMA: numpy
// evaluates one ufunc per operation, so this reproduces its results bit for bit.
//
// Layout: latents [T, D] frame-major float64.  A group of `lpf` lanes owns one frame
// (lpf = D/2 rounded up to a power of two, <= 32), each lane two adjacent channels
// (16-byte loads), so a D=64 frame is one fully coalesced 512-byte warp access per
// operand; the cfg-rescale norms are in-register shuffles over the group.
#include "rf_common.cuh"

namespace rf {

constexpr int kTickMaxRows = 32;
constexpr int kTickMaxGroups = 4;  // channel groups of 64 per lane -> D <= 256

// The rows travel as kernel parameters, sized to the launch (4, 8 or 32 rows): the launch
// cost grows with the parameter block (7.7 KB at 32 rows), and a tick has `depth` rows.
template <int CAP>
struct TickBatchT {
    int count;
    rf_row rows[CAP];
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ double curve_or(const double *c, int64_t f, double dflt) {
    return c ? c[f] : dflt;
}

// One element of the fused step; returns the new x and the guided output (for the
// rescale pass the caller needs the pre-rescale `out` and `vc`).
struct ElemVel {
    double vc;   // positive (blended) velocity
    double out;  // guided velocity before rescale
};

__device__ __forceinline__ double toy_velocity(double x, double x0p, double style, double t,
                                               const double *nm, double jt, int64_t i) {
    double x0 = dadd(x0p, style);
    double v = ddiv(dsub(x, x0), t);
    if (nm) v = dadd(v, dmul(jt, nm[i]));
    return v;
}

__device__ __forceinline__ ElemVel velocity_elem(const rf_row &R, const double *__restrict__ style,
                                                 double x, int64_t f, int64_t i) {
    const double t = R.t_curr;
    const bool cond_v = (R.flags & RF_ROWF_COND_V) != 0;
    const bool f32 = (R.flags & RF_ROWF_V_F32) != 0;
    // a given velocity (DiT output: float32, or a float64 seam input)
    auto given = [&](const double *p) -> double {
        double g = f32 ? (double)reinterpret_cast<const float *>(p)[i] : p[i];
        // shared style offset in x0 space for a velocity model: x0' = (x - v t) + style
        if (R.flags & RF_ROWF_STYLE_V) g = dsub(g, ddiv(style[i], t));
        return g;
    };
    double v;
    if (R.n_cond == 1) {
        v = cond_v ? given(R.cond_x0[0])
                   : toy_velocity(x, R.cond_x0[0][i], style[i], t, R.noise_model, R.jitter_t, i);
    } else {
        double acc = 0.0, tot = 0.0;
        for (int k = 0; k < R.n_cond; ++k) {
            double vk = cond_v ? given(R.cond_x0[k])
                               : toy_velocity(x, R.cond_x0[k][i], style[i], t, R.noise_model,
                                              R.jitter_t, i);
            double w = curve_or(R.cond_w[k], f, 1.0);
            acc = dadd(acc, dmul(w, vk));
            tot = dadd(tot, w);
        }
        v = ddiv(acc, tot);
    }
    ElemVel ev;
    ev.vc = v;
    ev.out = v;
    if (R.neg_kind == RF_NEG_NONE) return ev;
    double neg;
    if (R.neg_kind == RF_NEG_UNCOND) {
        double vu = (R.flags & RF_ROWF_UNCOND_V)
                        ? given(R.uncond_x0)
                        : toy_velocity(x, R.uncond_x0[i], style[i], t, R.noise_model, R.jitter_t, i);
        if (R.flags & RF_ROWF_WRITE_RESIDUAL) {
            double res = dsub(v, vu);
            R.residual[i] = res;
            neg = dsub(v, res);
        } else {
            neg = vu;
        }
    } else if (R.neg_kind == RF_NEG_RESIDUAL) {
        neg = dsub(v, R.residual[i]);
    } else {  // RF_NEG_PREV
        neg = R.prev_positive[i];
    }
    if (R.flags & RF_ROWF_WRITE_PREV) R.prev_positive[i] = v;
    double delta = dsub(v, neg);
    const double *apg = R.curves[RF_CURVE_APG];
    if (apg) {
        double m = (R.flags & RF_ROWF_MOMENTUM_INIT) ? 0.0 : R.momentum[i];
        m = dadd(dmul(apg[f], m), delta);
        R.momentum[i] = m;
        delta = m;
    }
    double scale = curve_or(R.curves[RF_CURVE_GUIDANCE], f, 1.0);
    ev.out = dadd(v, dmul(dsub(scale, 1.0), delta));
    return ev;
}

__device__ __forceinline__ double morph(const rf_row &R, double x0p, int64_t f, int64_t i) {
    double a = curve_or(R.curves[RF_CURVE_X0_STRENGTH], f, 1.0);
    return dadd(dmul(dsub(1.0, a), x0p), dmul(a, R.x0_target[i]));
}

__device__ __forceinline__ double solve_elem(const rf_row &R, double x, double v, int64_t f,
                                             int64_t i) {
    const double tc = R.t_curr, tn = R.t_next;
    if (R.solver == RF_SOLVER_SDE) {
        double x0p = dsub(x, dmul(v, tc));
        if (R.x0_target) x0p = morph(R, x0p, f, i);
        double n = R.noise_step[i];
        double tnn = dmul(tn, n);
        double omt = dsub(1.0, tn);
        double full = dadd(tnn, dmul(omt, x0p));
        if (!R.source) return full;
        double c = curve_or(R.curves[RF_CURVE_SDE], f, 1.0);
        double src = dadd(tnn, dmul(omt, R.source[i]));
        return dadd(dmul(c, full), dmul(dsub(1.0, c), src));
    }
    // ODE
    if (R.flags & RF_ROWF_ODE_MORPH) {
        double x0p = dsub(x, dmul(v, tc));
        v = ddiv(dsub(x, morph(R, x0p, f, i)), tc);
    }
    const double *vs = R.curves[RF_CURVE_VSCALE];
    if (vs) v = dmul(vs[f], v);
    double xn = dadd(x, dmul(v, dsub(tn, tc)));
    if (R.noise_step) xn = dadd(xn, dmul(R.curves[RF_CURVE_ODE_NOISE][f], R.noise_step[i]));
    return xn;
}

// Sum of squares over one frame's channels.  numpy's np.linalg.norm(axis=1) reduces
// each row with pairwise summation; here the order is a fixed shuffle tree, so the
// rescale factor is deterministic but may differ from numpy in the last ulp.
template <int LPF>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int off = LPF / 2; off > 0; off >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// The common row (one condition, no guidance, SDE step, no morph target) runs in its own
// lean kernel: the same operations in the same order as velocity_elem + solve_elem, on
// channel PAIRS (16-byte loads; 8-byte for fp32 velocities) indexed flat over the row, every
// operand of a thread's PPT pairs loaded before any arithmetic.  Split from the general
// kernel because register allocation is per kernel: the general path's 80 registers left
// 3 blocks per SM and 1.7 waves for the common case, which is HBM-bound and wants the whole
// launch resident in one wave with every load in flight (bench.py toy_path.solver_roofline).
__host__ __device__ inline bool fast_row(const rf_row &R, int64_t D) {
    const uintptr_t al = (uintptr_t)R.x | (uintptr_t)R.cond_x0[0] | (uintptr_t)R.noise_step |
                         (uintptr_t)R.source | (uintptr_t)R.noise_model;
    const uintptr_t need = (R.flags & RF_ROWF_V_F32) ? 7 : 15;
    return R.n_cond == 1 && R.neg_kind == RF_NEG_NONE && R.solver == RF_SOLVER_SDE && !R.x0_target &&
           !R.v_out && !(R.flags & RF_ROWF_NO_STEP) && R.x && R.noise_step && (D % 2) == 0 &&
           ((((uintptr_t)R.x | (uintptr_t)R.noise_step | (uintptr_t)R.source | (uintptr_t)R.noise_model) & 15) == 0) &&
           ((al & need) == 0);
}

// the fields of a fast row (88 bytes instead of rf_row's 248: a smaller parameter block)
struct FastRow {
    double *x;
    const void *v;             // cond_x0[0]: velocity (fp32 / fp64) or the toy x0 partial
    const double *nm;          // model noise or null
    const double *n;           // SDE noise
    const double *src;         // source or null
    const double *csde;        // per-frame SDE blend curve or null (= 1)
    double tc, tn, jt;
    int32_t flags;
};
template <int CAP>
struct FastBatchT {
    int count;
    uint32_t half_d;           // channel pairs per frame
    uint32_t pairs;            // channel pairs per row (T * D / 2)
    FastRow rows[CAP];
};

__device__ __forceinline__ double2 ld2(const double *p) { return __ldg((const double2 *)p); }

// One channel pair per thread, <= 64 registers (4 blocks of 256 per SM): 752 blocks for a
// config-2 tick, one wave.  Measured equal within noise to 2 pairs per thread (73 registers,
// 3 blocks per SM), 128-thread blocks and <= 40 registers; 4 pairs per thread +22%
// (profiles/r2_solver.txt).  The launch is latency-bound at this size (21.5 MB algorithmic,
// 11.5 MB from DRAM: the source, x0 table and style offset are shared by the rows).
constexpr int kFastThreads = 256;
constexpr int kFastPPT = 1;    // channel pairs per thread
constexpr int kFastMinBlocks = 4;

template <int CAP>
__global__ void __launch_bounds__(kFastThreads, kFastMinBlocks)
rf_tick_fast_kernel(const __grid_constant__ FastBatchT<CAP> B, const double *__restrict__ style) {
    pdl_wait();     // programmatic dependent launch: the prologue overlaps the previous kernel's tail
    pdl_launch();
    const FastRow &R = B.rows[blockIdx.y];
    const bool cond_v = (R.flags & RF_ROWF_COND_V) != 0, v32 = (R.flags & RF_ROWF_V_F32) != 0;
    const bool sty = !cond_v || (R.flags & RF_ROWF_STYLE_V);
    double2 x[kFastPPT], vg[kFastPPT], st[kFastPPT], nm[kFastPPT], n[kFastPPT], src[kFastPPT];
    double c[kFastPPT];
    uint32_t p[kFastPPT];
#pragma unroll
    for (int k = 0; k < kFastPPT; ++k) {
        p[k] = (blockIdx.x * kFastPPT + k) * kFastThreads + threadIdx.x;
        if (p[k] >= B.pairs) continue;
        const uint32_t i = 2 * p[k];
        x[k] = *(const double2 *)(R.x + i);
        if (cond_v && v32) {
            const float2 w = __ldg((const float2 *)R.v + p[k]);
            vg[k] = make_double2((double)w.x, (double)w.y);
        } else {
            vg[k] = ld2((const double *)R.v + i);
        }
        st[k] = sty ? ld2(style + i) : make_double2(0.0, 0.0);
        nm[k] = R.nm ? ld2(R.nm + i) : make_double2(0.0, 0.0);
        n[k] = ld2(R.n + i);
        src[k] = R.src ? ld2(R.src + i) : make_double2(0.0, 0.0);
        c[k] = (R.src && R.csde) ? __ldg(R.csde + p[k] / B.half_d) : 1.0;
    }
    const double tc = R.tc, tn = R.tn;
#pragma unroll
    for (int k = 0; k < kFastPPT; ++k) {
        if (p[k] >= B.pairs) continue;
        const double xv[2] = {x[k].x, x[k].y}, gv[2] = {vg[k].x, vg[k].y}, sv[2] = {st[k].x, st[k].y},
                     nmv[2] = {nm[k].x, nm[k].y}, nv[2] = {n[k].x, n[k].y}, srcv[2] = {src[k].x, src[k].y};
        double out[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double v;
            if (cond_v) {
                v = gv[e];
                if (R.flags & RF_ROWF_STYLE_V) v = dsub(v, ddiv(sv[e], tc));
            } else {   // toy_velocity
                const double x0 = dadd(gv[e], sv[e]);
                v = ddiv(dsub(xv[e], x0), tc);
                if (R.nm) v = dadd(v, dmul(R.jt, nmv[e]));
            }
            // solve_elem, SDE, no morph
            const double x0pe = dsub(xv[e], dmul(v, tc));
            const double tnn = dmul(tn, nv[e]);
            const double omt = dsub(1.0, tn);
            const double full = dadd(tnn, dmul(omt, x0pe));
            if (!R.src) {
                out[e] = full;
            } else {
                const double sr = dadd(tnn, dmul(omt, srcv[e]));
                out[e] = dadd(dmul(c[k], full), dmul(dsub(1.0, c[k]), sr));
            }
        }
        *(double2 *)(R.x + 2 * p[k]) = make_double2(out[0], out[1]);
    }
}

template <int LPF, int CAP>
__global__ void __launch_bounds__(256)
rf_tick_kernel(const __grid_constant__ TickBatchT<CAP> B, int64_t T, int64_t D, const double *__restrict__ style) {
    pdl_wait();
    pdl_launch();
    const rf_row &R = B.rows[blockIdx.y];
    const int lane = threadIdx.x & 31;
    constexpr int FPW = 32 / LPF;  // frames per warp step
    const int sub = lane / LPF, gl = lane % LPF;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const bool rescale = R.neg_kind != RF_NEG_NONE && R.curves[RF_CURVE_RESCALE] != nullptr;
    for (int64_t f0 = wid * FPW; f0 < T; f0 += warps_total * FPW) {
        const int64_t f = f0 + sub;
        const bool live = f < T;
        double vcs[kTickMaxGroups][2], outs[kTickMaxGroups][2], xs[kTickMaxGroups][2];
        double ss_out = 0.0, ss_pos = 0.0;
#pragma unroll
        for (int g = 0; g < kTickMaxGroups; ++g) {
            const int64_t c = (int64_t)g * 2 * LPF + 2 * gl;
            if (!live || c >= D) continue;
            const int64_t i = f * D + c;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (c + e >= D) continue;
                double x = R.x ? R.x[i + e] : 0.0;
                ElemVel ev = velocity_elem(R, style, x, f, i + e);
                xs[g][e] = x;
                vcs[g][e] = ev.vc;
                outs[g][e] = ev.out;
                if (rescale) {
                    ss_out = dadd(ss_out, dmul(ev.out, ev.out));
                    ss_pos = dadd(ss_pos, dmul(ev.vc, ev.vc));
                }
            }
        }
        double factor = 1.0;
        if (rescale) {
            ss_out = group_sum<LPF>(ss_out);
            ss_pos = group_sum<LPF>(ss_pos);
            if (live) {
                double no = sqrt(ss_out), np_ = sqrt(ss_pos);
                double keep = R.curves[RF_CURVE_RESCALE][f];
                double blended = dadd(dmul(keep, no), dmul(dsub(1.0, keep), np_));
                factor = no > 0.0 ? ddiv(blended, no) : 1.0;
            }
        }
#pragma unroll
        for (int g = 0; g < kTickMaxGroups; ++g) {
            const int64_t c = (int64_t)g * 2 * LPF + 2 * gl;
            if (!live || c >= D) continue;
            const int64_t i = f * D + c;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (c + e >= D) continue;
                double v = rescale ? dmul(outs[g][e], factor) : outs[g][e];
                if (R.v_out) R.v_out[i + e] = v;
                if (!(R.flags & RF_ROWF_NO_STEP)) R.x[i + e] = solve_elem(R, xs[g][e], v, f, i + e);
            }
        }
    }
}

template <int LPF, int CAP>
static int launch_tick(const TickBatchT<CAP> &B, int64_t T, int64_t D, const double *style,
                       cudaStream_t st) {
    constexpr int FPW = 32 / LPF;
    const int warps_per_block = 8;
    int64_t frames_per_block = (int64_t)warps_per_block * FPW;
    int64_t bx = (T + frames_per_block - 1) / frames_per_block;
    // keep >= ~2 waves over the SMs across all rows without oversubscribing tiny rows
    if (bx < 1) bx = 1;
    dim3 grid((unsigned)bx, (unsigned)B.count);
    RF_TRY_CUDA(launch_pdl(rf_tick_kernel<LPF, CAP>, grid, dim3(warps_per_block * 32), 0, st, B, T, D, style));
    RF_TRY_LAUNCH("rf_tick_kernel");
    return RF_OK;
}

template <int CAP>
static int launch_rows(const rf_row *rows, int n, int lpf, int64_t T, int64_t D, const double *style,
                       cudaStream_t st) {
    TickBatchT<CAP> B;
    B.count = n;
    for (int r = 0; r < n; ++r) B.rows[r] = rows[r];
    switch (lpf) {
        case 1: return launch_tick<1>(B, T, D, style, st);
        case 2: return launch_tick<2>(B, T, D, style, st);
        case 4: return launch_tick<4>(B, T, D, style, st);
        case 8: return launch_tick<8>(B, T, D, style, st);
        case 16: return launch_tick<16>(B, T, D, style, st);
        default: return launch_tick<32>(B, T, D, style, st);
    }
}

template <int CAP>
static int launch_fast(const FastRow *rows, int n, int64_t T, int64_t D, const double *style, cudaStream_t st) {
    FastBatchT<CAP> B;
    B.count = n;
    B.half_d = (uint32_t)(D / 2);
    B.pairs = (uint32_t)(T * D / 2);
    for (int r = 0; r < n; ++r) B.rows[r] = rows[r];
    const unsigned bx = (B.pairs + kFastThreads * kFastPPT - 1) / (kFastThreads * kFastPPT);
    RF_TRY_CUDA(launch_pdl(rf_tick_fast_kernel<CAP>, dim3(bx, (unsigned)n), dim3(kFastThreads), 0, st, B, style));
    RF_TRY_LAUNCH("rf_tick_fast_kernel");
    return RF_OK;
}

}  // namespace rf

using namespace rf;

extern "C" int rf_tick_solve(const rf_row *rows, int count, int64_t frames, int64_t channels,
                             const double *style_offset, void *stream) {
    if (count <= 0) return RF_OK;
    if (!rows || !style_offset || frames <= 0 || channels <= 0) {
        set_error("rf_tick_solve: bad arguments");
        return RF_EINVAL;
    }
    if (channels > 2 * 32 * kTickMaxGroups) {
        set_error("rf_tick_solve: channels %lld > %d", (long long)channels, 2 * 32 * kTickMaxGroups);
        return RF_EINVAL;
    }
    for (int r = 0; r < count; ++r) {
        const rf_row &R = rows[r];
        const bool velocity_only = (R.flags & RF_ROWF_NO_STEP) != 0;
        if ((!R.x && !velocity_only) || (velocity_only && !R.v_out) || R.n_cond < 1 ||
            R.n_cond > RF_MAX_COND || (!(R.t_curr > 0.0) && !(R.flags & RF_ROWF_COND_V))) {
            set_error("rf_tick_solve: bad row %d", r);
            return RF_EINVAL;
        }
        for (int k = 0; k < R.n_cond; ++k)
            if (!R.cond_x0[k]) {
                set_error("rf_tick_solve: row %d missing cond_x0[%d]", r, k);
                return RF_EINVAL;
            }
        if (!velocity_only && R.solver == RF_SOLVER_SDE && !R.noise_step) {
            set_error("rf_tick_solve: row %d sde without noise", r);
            return RF_EINVAL;
        }
        if (R.solver == RF_SOLVER_ODE && R.noise_step && !R.curves[RF_CURVE_ODE_NOISE]) {
            set_error("rf_tick_solve: row %d ode noise without curve", r);
            return RF_EINVAL;
        }
        if (!(R.flags & RF_ROWF_COND_V) && !R.x) {
            set_error("rf_tick_solve: row %d toy velocity needs x", r);
            return RF_EINVAL;
        }
        if ((R.flags & RF_ROWF_STYLE_V) && !(R.t_curr > 0.0)) {
            set_error("rf_tick_solve: row %d style offset on a velocity needs t_curr > 0", r);
            return RF_EINVAL;
        }
        if (R.neg_kind == RF_NEG_UNCOND && !R.uncond_x0) {
            set_error("rf_tick_solve: row %d guidance without uncond_x0", r);
            return RF_EINVAL;
        }
        if (R.curves[RF_CURVE_APG] && R.neg_kind != RF_NEG_NONE && !R.momentum) {
            set_error("rf_tick_solve: row %d apg without momentum buffer", r);
            return RF_EINVAL;
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    int64_t half = (channels + 1) / 2;
    int lpf = 1;
    while (lpf < half && lpf < 32) lpf <<= 1;
    // common rows to the lean kernel, the rest (guidance, multi-condition, ODE, morph,
    // velocity-only) to the general one; rows are independent, so the split keeps results
    rf_row general[kTickMaxRows];
    FastRow fast[kTickMaxRows];
    int ng = 0, nf = 0;
    for (int r = 0; r <= count; ++r) {
        if (r < count) {
            const rf_row &R = rows[r];
            if (fast_row(R, channels)) {
                FastRow &F = fast[nf++];
                F.x = R.x;
                F.v = R.cond_x0[0];
                F.nm = R.noise_model;
                F.n = R.noise_step;
                F.src = R.source;
                F.csde = R.curves[RF_CURVE_SDE];
                F.tc = R.t_curr;
                F.tn = R.t_next;
                F.jt = R.jitter_t;
                F.flags = R.flags;
            } else {
                general[ng++] = R;
            }
        }
        const bool last = r == count;
        if (nf && (nf == kTickMaxRows || last)) {
            const int rc = nf <= 4 ? launch_fast<4>(fast, nf, frames, channels, style_offset, st)
                         : nf <= 8 ? launch_fast<8>(fast, nf, frames, channels, style_offset, st)
                                   : launch_fast<kTickMaxRows>(fast, nf, frames, channels, style_offset, st);
            if (rc) return rc;
            nf = 0;
        }
        if (ng && (ng == kTickMaxRows || last)) {
            const int rc = ng <= 4 ? launch_rows<4>(general, ng, lpf, frames, channels, style_offset, st)
                         : ng <= 8 ? launch_rows<8>(general, ng, lpf, frames, channels, style_offset, st)
                                   : launch_rows<kTickMaxRows>(general, ng, lpf, frames, channels, style_offset, st);
            if (rc) return rc;
            ng = 0;
        }
    }
    return RF_OK;
}
