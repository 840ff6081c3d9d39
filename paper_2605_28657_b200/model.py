"""The velocity model slot: the closed-form toy flow model, on the device.

Mirrors reference ``pkg/src/ringflow/model.py`` (public names :24).  The toy model's
"weights" are per-prompt harmonic pattern tables (model.py:104-121): their amplitudes
and phases are drawn on the GPU with the bit-exact keyed noise, and the [T, C] table is
evaluated once per (kind, prompt) at setup -- on the host with numpy's sin, so the
table bytes equal the reference's -- then kept resident in HBM.  Per tick, velocities
are computed inside the fused solver kernel (csrc/rf_tick.cu) from the resident
x0 tables; ``velocity`` / ``x0_of`` below are seams that run the same kernels.

The ACE-Step-shape DiT that replaces this model for configs 2-5 is ``dit.py``.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np
import torch

from . import _device, _native
from .latents import NoiseSource, content_hash

__all__ = ["ConditionSet", "ModelWeights", "ToyFlowModel", "UNCOND_PROMPT"]

UNCOND_PROMPT = 0
PATTERN_HARMONICS = 4
HINT_SCALE = 0.45
TIMBRE_SCALE = 0.45


def _frozen_copy(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        a = x.detach().to("cpu", torch.float64).numpy().copy()
    else:
        a = np.array(x, dtype=np.float64, copy=True)
    a.setflags(write=False)
    return a


@dataclass(frozen=True)
class ConditionSet:
    """One frozen conditioning bundle (model.py:33-64)."""

    prompt_hash: int
    hint_strength: float = 0.0
    timbre_strength: float = 0.0
    source: Optional[object] = None       # [T, D] numpy array or tensor
    weight_curve: Optional[object] = None  # [T] or None (uniform)
    _cache: dict = field(default_factory=dict, init=False, repr=False, compare=False, hash=False)

    def __post_init__(self):
        if not 0.0 <= self.hint_strength <= 1.0:
            raise ValueError("hint_strength must be in [0, 1]")
        if not 0.0 <= self.timbre_strength <= 1.0:
            raise ValueError("timbre_strength must be in [0, 1]")
        # The bundle is frozen in content too: ``source`` / ``weight_curve`` are copied at
        # construction (read-only host arrays), so the cached content key and device copies
        # below can never go stale if the caller later mutates the array it passed in.
        # (The reference re-hashes on every call, model.py:52-61; with an immutable copy the
        # cached key is the same value.)
        for name in ("source", "weight_curve"):
            val = getattr(self, name)
            if val is not None:
                object.__setattr__(self, name, _frozen_copy(val))

    def content_key(self) -> int:
        """Hash of the conditioning content; keys the noise streams (model.py:53-61)."""
        key = self._cache.get("content_key")
        if key is None:
            key = content_hash(self.prompt_hash, self.hint_strength, self.timbre_strength,
                               self.source, self.weight_curve)
            self._cache["content_key"] = key
        return key

    def with_source(self, source) -> "ConditionSet":
        return replace(self, source=source)

    def source_device(self, dev=None) -> Optional[torch.Tensor]:
        if self.source is None:
            return None
        t = self._cache.get("source_dev")
        if t is None:
            t = _device.to_device_f64(self.source, dev)
            self._cache["source_dev"] = t
        return t

    def weight_device(self, dev=None) -> Optional[torch.Tensor]:
        if self.weight_curve is None:
            return None
        t = self._cache.get("weight_dev")
        if t is None:
            t = _device.to_device_f64(self.weight_curve, dev)
            self._cache["weight_dev"] = t
        return t


class ModelWeights:
    """Shared mutable style offset added to every x0 (model.py:67-88); lives in HBM."""

    def __init__(self, style_offset, version: int = 0):
        self._dev = _device.to_device_f64(style_offset)
        self.version = version

    @classmethod
    def zeros(cls, shape) -> "ModelWeights":
        w = cls.__new__(cls)
        w._dev = torch.zeros(tuple(shape), dtype=torch.float64, device=_device.device())
        w.version = 0
        return w

    @property
    def style_offset(self) -> np.ndarray:
        return self._dev.cpu().numpy()

    @property
    def device_offset(self) -> torch.Tensor:
        return self._dev

    def swap_offset(self, offset) -> None:
        if tuple(offset.shape) != tuple(self._dev.shape):
            raise ValueError(f"offset shape {tuple(offset.shape)} != {tuple(self._dev.shape)}")
        # a fresh buffer: kernels already enqueued keep reading the old version
        self._dev = _device.to_device_f64(offset).clone()
        self.version += 1


class ToyFlowModel:
    """Deterministic velocity oracle over [frames, channels] latents (model.py:91-152)."""

    def __init__(self, frames: int, channels: int, perturbation: float = 0.0):
        self.frames = frames
        self.channels = channels
        self.perturbation = perturbation
        self._patterns: dict = {}
        self._partials: dict = {}

    @property
    def shape(self):
        return (self.frames, self.channels)

    def pattern_device(self, kind: str, prompt_hash: int) -> torch.Tensor:
        key = (kind, prompt_hash)
        hit = self._patterns.get(key)
        if hit is not None:
            return hit
        rng = NoiseSource(seed=prompt_hash, stream=content_hash("pattern", kind))
        amps = rng.normal(0, "amps", (PATTERN_HARMONICS, self.channels))
        phases = 2.0 * np.pi * rng.uniform(0, "phases", (PATTERN_HARMONICS, self.channels))
        t = (np.arange(self.frames, dtype=np.float64) + 0.5) / self.frames
        table = np.zeros(self.shape)
        for k in range(PATTERN_HARMONICS):
            table += amps[k][None, :] * np.sin(2.0 * np.pi * (k + 1) * t[:, None] + phases[k][None, :])
        table /= np.sqrt(PATTERN_HARMONICS)
        dev = _device.to_device_f64(table)
        self._patterns[key] = dev
        return dev

    def pattern(self, kind: str, prompt_hash: int) -> np.ndarray:
        out = self.pattern_device(kind, prompt_hash).cpu().numpy()
        out.setflags(write=False)
        return out

    def x0_partial(self, cond: ConditionSet) -> torch.Tensor:
        """base + (h*0.45)*hint + (tau*0.45)*timbre on the device (style added per step)."""
        key = (cond.prompt_hash, cond.hint_strength, cond.timbre_strength)
        hit = self._partials.get(key)
        if hit is not None:
            return hit
        base = self.pattern_device("base", cond.prompt_hash)
        hint = self.pattern_device("hint", cond.prompt_hash) if cond.hint_strength != 0.0 else None
        timbre = self.pattern_device("timbre", cond.prompt_hash) if cond.timbre_strength != 0.0 else None
        out = torch.empty_like(base)
        lib = _native.load()
        _native.check(lib.rf_x0_compose(
            out.data_ptr(), base.data_ptr(), hint.data_ptr() if hint is not None else None,
            cond.hint_strength * HINT_SCALE, timbre.data_ptr() if timbre is not None else None,
            cond.timbre_strength * TIMBRE_SCALE, None, out.numel(), _device.current_stream_handle()),
            "rf_x0_compose")
        # cached and read from any pipeline's stream: complete it before handing it out
        torch.cuda.current_stream().synchronize()
        self._partials[key] = out
        return out

    def x0_of_device(self, cond: ConditionSet, weights: ModelWeights) -> torch.Tensor:
        part = self.x0_partial(cond)
        style = weights.device_offset
        out = torch.empty_like(part)
        lib = _native.load()
        _native.check(lib.rf_x0_compose(out.data_ptr(), part.data_ptr(), None, 0.0, None, 0.0,
                                        style.data_ptr(), out.numel(), _device.current_stream_handle()),
                      "rf_x0_compose")
        return out

    def x0_of(self, cond: ConditionSet, weights: ModelWeights) -> np.ndarray:
        return self.x0_of_device(cond, weights).cpu().numpy()

    def velocity_device(self, x_t, t: float, cond: ConditionSet, weights: ModelWeights,
                        rng: NoiseSource, step: int) -> torch.Tensor:
        if t <= 0.0:
            raise ValueError("velocity is undefined at t <= 0")
        from . import solver as _solver  # the fused kernel runs the velocity

        x = _device.to_device_f64(x_t)
        noise = rng.normal_device(step, "model", tuple(x.shape)) if self.perturbation != 0.0 else None
        return _solver._run_velocity(
            x=x, t=t, conds=[(self.x0_partial(cond), None)], style=weights.device_offset,
            noise_model=noise, jitter_t=self.perturbation * t)

    def velocity(self, x_t, t: float, cond: ConditionSet, weights: ModelWeights,
                 rng: NoiseSource, step: int) -> np.ndarray:
        return self.velocity_device(x_t, t, cond, weights, rng, step).cpu().numpy()
