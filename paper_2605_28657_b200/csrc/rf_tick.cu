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

// The common row (one condition, no guidance, SDE step, no morph target): the same
// operations in the same order as velocity_elem + solve_elem, but every operand of a
// lane's two channels is fetched with one 16-byte (8-byte for fp32 velocities) load,
// all of them issued before any arithmetic, so a thread makes one memory round trip
// instead of a chain of dependent scalar loads.  The kernel is HBM-bound; this is what
// lets it approach the roofline (bench.py toy_path.solver_roofline).
__device__ __forceinline__ bool fast_row(const rf_row &R, int64_t D) {
    const uintptr_t al = (uintptr_t)R.x | (uintptr_t)R.cond_x0[0] | (uintptr_t)R.noise_step |
                         (uintptr_t)R.source | (uintptr_t)R.noise_model;
    const uintptr_t need = (R.flags & RF_ROWF_V_F32) ? 7 : 15;
    return R.n_cond == 1 && R.neg_kind == RF_NEG_NONE && R.solver == RF_SOLVER_SDE && !R.x0_target &&
           !R.v_out && !(R.flags & RF_ROWF_NO_STEP) && R.x && R.noise_step && (D % 2) == 0 &&
           ((((uintptr_t)R.x | (uintptr_t)R.noise_step | (uintptr_t)R.source | (uintptr_t)R.noise_model) & 15) == 0) &&
           ((al & need) == 0);
}

__device__ __forceinline__ double2 ld2(const double *p) { return __ldg((const double2 *)p); }

__device__ __forceinline__ void fast_pair(const rf_row &R, const double *__restrict__ style, int64_t f, int64_t i) {
    const double2 x = *(const double2 *)(R.x + i);
    const bool cond_v = (R.flags & RF_ROWF_COND_V) != 0;
    double2 vg = make_double2(0.0, 0.0), x0p = vg, st = vg, nm = vg, src = vg;
    if (cond_v) {
        if (R.flags & RF_ROWF_V_F32) {
            const float2 v32 = __ldg((const float2 *)R.cond_x0[0] + i / 2);
            vg = make_double2((double)v32.x, (double)v32.y);
        } else {
            vg = ld2(R.cond_x0[0] + i);
        }
        if (R.flags & RF_ROWF_STYLE_V) st = ld2(style + i);
    } else {
        x0p = ld2(R.cond_x0[0] + i);
        st = ld2(style + i);
        if (R.noise_model) nm = ld2(R.noise_model + i);
    }
    const double2 n = ld2(R.noise_step + i);
    if (R.source) src = ld2(R.source + i);
    const double c = R.source ? curve_or(R.curves[RF_CURVE_SDE], f, 1.0) : 1.0;
    const double tc = R.t_curr, tn = R.t_next;
    const double xv[2] = {x.x, x.y}, vgv[2] = {vg.x, vg.y}, x0v[2] = {x0p.x, x0p.y}, sv[2] = {st.x, st.y},
                 nmv[2] = {nm.x, nm.y}, nv[2] = {n.x, n.y}, srcv[2] = {src.x, src.y};
    double out[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        double v;
        if (cond_v) {
            v = vgv[e];
            if (R.flags & RF_ROWF_STYLE_V) v = dsub(v, ddiv(sv[e], tc));
        } else {   // toy_velocity
            const double x0 = dadd(x0v[e], sv[e]);
            v = ddiv(dsub(xv[e], x0), tc);
            if (R.noise_model) v = dadd(v, dmul(R.jitter_t, nmv[e]));
        }
        // solve_elem, SDE, no morph
        const double x0pe = dsub(xv[e], dmul(v, tc));
        const double tnn = dmul(tn, nv[e]);
        const double omt = dsub(1.0, tn);
        const double full = dadd(tnn, dmul(omt, x0pe));
        if (!R.source) {
            out[e] = full;
        } else {
            const double sr = dadd(tnn, dmul(omt, srcv[e]));
            out[e] = dadd(dmul(c, full), dmul(dsub(1.0, c), sr));
        }
    }
    *(double2 *)(R.x + i) = make_double2(out[0], out[1]);
}

template <int LPF, int CAP>
__global__ void __launch_bounds__(256)
rf_tick_kernel(const __grid_constant__ TickBatchT<CAP> B, int64_t T, int64_t D, const double *__restrict__ style) {
    const rf_row &R = B.rows[blockIdx.y];
    const int lane = threadIdx.x & 31;
    constexpr int FPW = 32 / LPF;  // frames per warp step
    const int sub = lane / LPF, gl = lane % LPF;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const bool rescale = R.neg_kind != RF_NEG_NONE && R.curves[RF_CURVE_RESCALE] != nullptr;
    if (fast_row(R, D)) {
        for (int64_t f0 = wid * FPW; f0 < T; f0 += warps_total * FPW) {
            const int64_t f = f0 + sub;
            if (f >= T) continue;
#pragma unroll
            for (int g = 0; g < kTickMaxGroups; ++g) {
                const int64_t c = (int64_t)g * 2 * LPF + 2 * gl;
                if (c < D) fast_pair(R, style, f, f * D + c);
            }
        }
        return;
    }

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
    rf_tick_kernel<LPF, CAP><<<grid, warps_per_block * 32, 0, st>>>(B, T, D, style);
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
    for (int r0 = 0; r0 < count; r0 += kTickMaxRows) {
        const int n = count - r0 < kTickMaxRows ? count - r0 : kTickMaxRows;
        const int rc = n <= 4 ? launch_rows<4>(rows + r0, n, lpf, frames, channels, style_offset, st)
                     : n <= 8 ? launch_rows<8>(rows + r0, n, lpf, frames, channels, style_offset, st)
                              : launch_rows<kTickMaxRows>(rows + r0, n, lpf, frames, channels, style_offset, st);
        if (rc) return rc;
    }
    return RF_OK;
}
