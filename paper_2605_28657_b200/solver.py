"""Per-step denoising math on the GPU: curves, guidance, SDE/ODE steps.

Mirrors reference ``pkg/src/ringflow/solver.py`` (public names :31-43).  Curve plumbing
(field table, clamping, sentinels; solver.py:45-115) is host bookkeeping on [T] vectors.
All latent arithmetic runs in the fused tick kernel ``rf_tick_solve``
(csrc/rf_tick.cu); the functions below are the reference's function seams, each
issuing one launch of that kernel with the velocities given as inputs, so the seams
and the pipeline share one implementation.  Results come back as numpy arrays (the
reference's return type); ``*_device`` variants return tensors.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _device, _native
from ._native import CURVE_INDEX
from .latents import NoiseSource, ShapeMismatchError

__all__ = [
    "CURVE_FIELDS",
    "CurveSet",
    "StepState",
    "MissingSourceError",
    "clamp_curve",
    "sentinel",
    "as_curve",
    "make_curves",
    "guided_velocity",
    "blend_conditions",
    "ode_step",
    "sde_step",
]

# name -> (kind, lo, hi); kind fixes the sentinel (mult: ones, add: zeros).  solver.py:48-56
CURVE_FIELDS = {
    "sde_denoise_curve": ("mult", 0.0, 1.0),
    "guidance_curve": ("mult", 0.0, 8.0),
    "velocity_scale": ("mult", 0.0, 4.0),
    "ode_noise_curve": ("add", 0.0, 1.0),
    "apg_momentum": ("add", -1.0, 1.0),
    "cfg_rescale_curve": ("mult", 0.0, 1.0),
    "x0_target_strength": ("mult", 0.0, 1.0),
}
RCFG_MODES = ("off", "full-cfg", "onetime-negative", "self-negative")


class MissingSourceError(ValueError):
    """An SDE step needed source latents (blend curve < 1 somewhere) but had none."""


def sentinel(name: str, frames: int) -> np.ndarray:
    return np.ones(frames) if CURVE_FIELDS[name][0] == "mult" else np.zeros(frames)


def clamp_curve(name: str, values, frames: int) -> np.ndarray:
    """Scalar-or-vector -> clipped float64 [frames] curve (solver.py:71-83)."""
    if name not in CURVE_FIELDS:
        raise KeyError(f"unknown curve field {name!r}")
    _, lo, hi = CURVE_FIELDS[name]
    if isinstance(values, torch.Tensor):
        values = values.detach().cpu().numpy()
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim == 0:
        arr = np.full(frames, float(arr))
    if arr.shape != (frames,):
        raise ShapeMismatchError(f"{name} must have shape ({frames},), got {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{name} contains non-finite entries")
    return np.clip(arr, lo, hi)


as_curve = clamp_curve


@dataclass(frozen=True)
class CurveSet:
    """The per-frame controls one solver step reads (solver.py:86-105)."""

    sde_denoise_curve: Optional[np.ndarray] = None
    guidance_curve: Optional[np.ndarray] = None
    velocity_scale: Optional[np.ndarray] = None
    ode_noise_curve: Optional[np.ndarray] = None
    apg_momentum: Optional[np.ndarray] = None
    cfg_rescale_curve: Optional[np.ndarray] = None
    x0_target_strength: Optional[np.ndarray] = None
    x0_target: Optional[object] = None
    guidance_enabled: bool = False
    rcfg_mode: str = "off"
    _cache: dict = field(default_factory=dict, init=False, repr=False, compare=False, hash=False)

    def __post_init__(self):
        if self.rcfg_mode not in RCFG_MODES:
            raise ValueError(f"rcfg_mode must be one of {RCFG_MODES}")
        if self.x0_target_strength is not None and self.x0_target is None:
            raise ValueError("x0_target_strength requires x0_target")
        # immutable content: array fields are read-only copies, so the device copies cached
        # below cannot go stale when the caller mutates what it passed in
        for name in tuple(CURVE_FIELDS) + ("x0_target",):
            val = getattr(self, name)
            if val is not None:
                if isinstance(val, torch.Tensor):
                    arr = val.detach().to("cpu", torch.float64).numpy().copy()
                else:
                    arr = np.array(val, dtype=np.float64, copy=True)
                arr.setflags(write=False)
                object.__setattr__(self, name, arr)

    def device(self, name: str) -> Optional[torch.Tensor]:
        """Resident device copy of a curve (or of x0_target)."""
        val = getattr(self, name)
        if val is None:
            return None
        t = self._cache.get(name)
        if t is None:
            t = _device.to_device_f64(val)
            self._cache[name] = t
        return t


def make_curves(frames: int, x0_target=None, guidance_enabled: bool = False,
                rcfg_mode: str = "off", **named) -> CurveSet:
    clamped = {n: clamp_curve(n, v, frames) for n, v in named.items() if v is not None}
    return CurveSet(x0_target=x0_target, guidance_enabled=guidance_enabled, rcfg_mode=rcfg_mode,
                    **clamped)


class DeviceState(torch.Tensor):
    """A device buffer of solver state that converts to a host numpy array on demand
    (``np.asarray(state.residual)``), as the reference's numpy state does (solver.py:118-134);
    the kernels use it in place on the device."""

    def __array__(self, dtype=None, copy=None):
        a = self.detach().as_subclass(torch.Tensor).cpu().numpy()
        return a if dtype is None else a.astype(dtype, copy=False)


def _state_buffer(like) -> torch.Tensor:
    return torch.empty_like(like).as_subclass(DeviceState)


@dataclass
class StepState:
    """Slot-owned solver scratch (solver.py:118-134); buffers live on the device."""

    steps_total: int
    step: int = 0
    momentum: Optional[torch.Tensor] = None
    residual: Optional[torch.Tensor] = None
    prev_positive: Optional[torch.Tensor] = None

    def in_refinement_half(self) -> bool:
        return self.step >= self.steps_total // 2


# ----------------------------------------------------------------- row assembly ----

def _p(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def curve_pointers(row: _native.RfRow, getter) -> None:
    for name, idx in CURVE_INDEX.items():
        row.curves[idx] = _p(getter(name))


def guidance_plan(mode: str, state: StepState, have_uncond: bool):
    """(neg_kind, flags) for one guided step, following solver.py:161-180."""
    if mode in ("off", "full-cfg"):
        if not have_uncond:
            raise ValueError("guidance requires a negative velocity each step")
        return _native.RF_NEG_UNCOND, 0
    if mode == "onetime-negative":
        if state.residual is None:
            if not have_uncond:
                raise ValueError("onetime-negative needs a negative at step 0")
            return _native.RF_NEG_UNCOND, _native.RF_ROWF_WRITE_RESIDUAL
        return _native.RF_NEG_RESIDUAL, 0
    if mode == "self-negative":
        if state.prev_positive is None:
            if not have_uncond:
                raise ValueError("self-negative needs a negative at step 0")
            return _native.RF_NEG_UNCOND, _native.RF_ROWF_WRITE_PREV
        return _native.RF_NEG_PREV, _native.RF_ROWF_WRITE_PREV
    raise ValueError(mode)


def prepare_guidance_state(row: _native.RfRow, state: StepState, curves_apg_present: bool,
                           like: torch.Tensor) -> None:
    """Allocate the slot's guidance buffers the kernel will write and wire pointers."""
    if row.flags & _native.RF_ROWF_WRITE_RESIDUAL:
        state.residual = _state_buffer(like)
    if row.flags & _native.RF_ROWF_WRITE_PREV and state.prev_positive is None:
        state.prev_positive = _state_buffer(like)
    if curves_apg_present:
        if state.momentum is None:
            state.momentum = _state_buffer(like)
            row.flags |= _native.RF_ROWF_MOMENTUM_INIT
    row.momentum = _p(state.momentum)
    row.residual = _p(state.residual)
    row.prev_positive = _p(state.prev_positive)


def launch_rows(rows, frames: int, channels: int, style: torch.Tensor) -> None:
    lib = _native.load()
    n = len(rows)
    if n == 0:
        return
    arr = (_native.RfRow * n)(*rows)
    _native.check(lib.rf_tick_solve(arr, n, frames, channels, style.data_ptr(),
                                    _device.current_stream_handle()), "rf_tick_solve")


_ZERO_STYLE: dict = {}


def _zero_style(shape, dev) -> torch.Tensor:
    key = (tuple(shape), dev.index)
    t = _ZERO_STYLE.get(key)
    if t is None:
        t = _ZERO_STYLE[key] = torch.zeros(tuple(shape), dtype=torch.float64, device=dev)
    return t


def _run_velocity(x, t, conds, style, noise_model, jitter_t) -> torch.Tensor:
    """Toy-model velocity (model.py:133-152) through the fused kernel, no state update."""
    out = torch.empty_like(x)
    row = _native.RfRow()
    row.x = x.data_ptr()
    row.noise_model = _p(noise_model)
    row.n_cond = len(conds)
    for k, (x0p, w) in enumerate(conds):
        row.cond_x0[k] = x0p.data_ptr()
        row.cond_w[k] = _p(w)
    row.v_out = out.data_ptr()
    row.t_curr = float(t)
    row.jitter_t = float(jitter_t)
    row.flags = _native.RF_ROWF_NO_STEP
    T, D = x.shape
    launch_rows([row], T, D, style)
    return out


# ------------------------------------------------------------------- the seams ----

def _dev_latent(a):
    return _device.to_device_f64(a)


def guided_velocity(v_cond, v_uncond, curves: CurveSet, state: StepState, step_index: int):
    """Classifier-free guidance with rcfg variants, APG and rescale (solver.py:141-201)."""
    vc = _dev_latent(v_cond)
    vu = None if v_uncond is None else _dev_latent(v_uncond)
    frames = vc.shape[0]
    neg_kind, flags = guidance_plan(curves.rcfg_mode, state, vu is not None)
    out = torch.empty_like(vc)
    row = _native.RfRow()
    row.cond_x0[0] = vc.data_ptr()
    row.n_cond = 1
    row.uncond_x0 = _p(vu)
    row.neg_kind = neg_kind
    row.flags = flags | _native.RF_ROWF_COND_V | _native.RF_ROWF_UNCOND_V | _native.RF_ROWF_NO_STEP
    row.v_out = out.data_ptr()
    row.t_curr = 1.0
    curve_pointers(row, curves.device)
    prepare_guidance_state(row, state, curves.apg_momentum is not None, vc)
    launch_rows([row], frames, vc.shape[1], _zero_style(vc.shape, vc.device))
    return out.cpu().numpy()


def blend_conditions(velocities: list, weights: list):
    """Per-frame convex combination sum(w_i v_i)/sum(w_i) (solver.py:204-227)."""
    if not velocities:
        raise ValueError("at least one condition velocity required")
    if len(velocities) != len(weights):
        raise ValueError("one weight curve per velocity required")
    if len(velocities) == 1:
        return velocities[0]
    if len(velocities) > _native.RF_MAX_COND:
        raise NotImplementedError(f"at most {_native.RF_MAX_COND} blended conditions per row")
    ws = [np.asarray(w.cpu() if isinstance(w, torch.Tensor) else w, dtype=np.float64) for w in weights]
    for w in ws:
        if np.any(w < 0.0):
            raise ValueError("condition weights must be nonnegative")
    total = np.zeros_like(ws[0])
    for w in ws:
        total += w
    if np.any(total <= 0.0):
        raise ValueError("condition weights sum to zero at some frame")
    vs = [_dev_latent(v) for v in velocities]
    wd = [_device.to_device_f64(w) for w in ws]
    out = torch.empty_like(vs[0])
    row = _native.RfRow()
    row.n_cond = len(vs)
    for k in range(len(vs)):
        row.cond_x0[k] = vs[k].data_ptr()
        row.cond_w[k] = wd[k].data_ptr()
    row.flags = _native.RF_ROWF_COND_V | _native.RF_ROWF_NO_STEP
    row.v_out = out.data_ptr()
    row.t_curr = 1.0
    launch_rows([row], vs[0].shape[0], vs[0].shape[1], _zero_style(vs[0].shape, vs[0].device))
    return out.cpu().numpy()


def _check_shapes(x_t, v) -> None:
    if tuple(x_t.shape) != tuple(v.shape):
        raise ShapeMismatchError(
            f"latent/velocity shape mismatch: {tuple(x_t.shape)} vs {tuple(v.shape)}")


def ode_step(x_t, v, t_curr: float, t_next: float, curves: CurveSet, rng: NoiseSource,
             state: Optional[StepState] = None):
    """Euler step with velocity_scale and additive ode noise (solver.py:241-270)."""
    if t_next >= t_curr:
        raise ValueError(f"timesteps must decrease: {t_curr} -> {t_next}")
    _check_shapes(x_t, v)
    x = _dev_latent(x_t).clone()
    vd = _dev_latent(v)
    row = _native.RfRow()
    row.x = x.data_ptr()
    row.cond_x0[0] = vd.data_ptr()
    row.n_cond = 1
    row.solver = _native.RF_SOLVER_ODE
    row.flags = _native.RF_ROWF_COND_V
    row.t_curr, row.t_next = float(t_curr), float(t_next)
    curve_pointers(row, curves.device)
    if state is not None and curves.x0_target is not None and state.in_refinement_half():
        row.flags |= _native.RF_ROWF_ODE_MORPH
        row.x0_target = curves.device("x0_target").data_ptr()
    noise = None
    if curves.ode_noise_curve is not None:
        step = 0 if state is None else state.step
        noise = rng.normal_device(step, "ode", tuple(x.shape))
        row.noise_step = noise.data_ptr()
    launch_rows([row], x.shape[0], x.shape[1], _zero_style(x.shape, x.device))
    return x.cpu().numpy()


def sde_step(x_t, v, t_curr: float, t_next: float, source, curves: CurveSet, state: StepState,
             rng: NoiseSource):
    """SDE re-noise with per-frame source blending (solver.py:273-306)."""
    if t_next >= t_curr:
        raise ValueError(f"timesteps must decrease: {t_curr} -> {t_next}")
    _check_shapes(x_t, v)
    curve = curves.sde_denoise_curve
    if source is None:
        if curve is not None and np.any(curve < 1.0):
            raise MissingSourceError("sde_denoise_curve < 1 requires source latents")
    elif tuple(source.shape) != tuple(x_t.shape):
        raise ShapeMismatchError(f"source shape {tuple(source.shape)} != {tuple(x_t.shape)}")
    x = _dev_latent(x_t).clone()
    vd = _dev_latent(v)
    src = None if source is None else _dev_latent(source)
    noise = rng.normal_device(state.step, "sde", tuple(x.shape))
    row = _native.RfRow()
    row.x = x.data_ptr()
    row.cond_x0[0] = vd.data_ptr()
    row.n_cond = 1
    row.solver = _native.RF_SOLVER_SDE
    row.flags = _native.RF_ROWF_COND_V
    row.t_curr, row.t_next = float(t_curr), float(t_next)
    row.noise_step = noise.data_ptr()
    row.source = _p(src)
    curve_pointers(row, curves.device)
    if curves.x0_target is not None and state.in_refinement_half():
        row.x0_target = curves.device("x0_target").data_ptr()
    launch_rows([row], x.shape[0], x.shape[1], _zero_style(x.shape, x.device))
    return x.cpu().numpy()
