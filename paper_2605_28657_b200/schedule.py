"""Sigma ladders for ring slots (host bookkeeping).

Behaviour follows reference ``pkg/src/ringflow/schedule.py`` (ladder :48-75, cache
:78-98, migration :101-116): sigma_i = d * s*u / (1 + (s-1)*u) with u = 1 - i/S, the
two ends pinned to d and 0, id = blake2b-6 over the float64 bytes of the ladder and
the shift.  A ladder is S+1 host doubles; the tick only gathers (sigma[k],
sigma[k+1]) per row into its launch descriptor, so indexing stays bit-exact and
nothing here touches the device.
"""
from __future__ import annotations

import hashlib
from typing import Dict, Tuple

import numpy as np

__all__ = [
    "TimestepSchedule",
    "ScheduleCache",
    "ScheduleMismatchError",
    "build_schedule",
    "migrate_schedule",
]

DENOISE_QUANTUM = 1e-6


class ScheduleMismatchError(ValueError):
    """Migration refused: the two ladders have different step counts."""


class TimestepSchedule:
    """Immutable ladder + identity.  Attribute names match the reference dataclass."""

    __slots__ = ("sigmas", "denoise", "steps", "shift", "schedule_id")

    def __init__(self, sigmas: np.ndarray, denoise: float, steps: int, shift: float,
                 schedule_id: str):
        sigmas.setflags(write=False)
        object.__setattr__(self, "sigmas", sigmas)
        object.__setattr__(self, "denoise", denoise)
        object.__setattr__(self, "steps", steps)
        object.__setattr__(self, "shift", shift)
        object.__setattr__(self, "schedule_id", schedule_id)

    def __setattr__(self, name, value):
        raise AttributeError("TimestepSchedule is immutable")

    def __repr__(self) -> str:
        return (f"TimestepSchedule(id={self.schedule_id}, denoise={self.denoise}, "
                f"steps={self.steps}, shift={self.shift})")

    def pair(self, k: int) -> Tuple[float, float]:
        """(t_curr, t_next) for step k, as Python floats (exact float64 values)."""
        return float(self.sigmas[k]), float(self.sigmas[k + 1])


def _ladder(denoise: float, steps: int, shift: float) -> np.ndarray:
    # Same float64 operation sequence as the reference so the bytes (and ids) agree.
    u = 1.0 - np.arange(steps + 1, dtype=np.float64) / steps
    warped = shift * u / (1.0 + (shift - 1.0) * u)
    ladder = denoise * warped
    ladder[0], ladder[-1] = denoise, 0.0
    return ladder


def build_schedule(denoise: float, steps: int, shift: float = 3.0) -> TimestepSchedule:
    checks = (
        (0.0 < denoise <= 1.0, f"denoise must be in (0, 1], got {denoise}"),
        (steps >= 1, f"steps must be >= 1, got {steps}"),
        (shift > 0.0, f"shift must be > 0, got {shift}"),
    )
    for ok, msg in checks:
        if not ok:
            raise ValueError(msg)
    ladder = _ladder(denoise, steps, shift)
    if not bool((ladder[1:] < ladder[:-1]).all()):
        raise AssertionError("schedule sigmas must decrease strictly")
    h = hashlib.blake2b(ladder.tobytes(), digest_size=6)
    h.update(np.float64(shift).tobytes())
    return TimestepSchedule(ladder, denoise, steps, shift, h.hexdigest())


class ScheduleCache:
    """Session cache; equal (quantised) strengths share one ladder object. Never evicts."""

    def __init__(self):
        self._entries: Dict[tuple, TimestepSchedule] = {}

    def get(self, denoise: float, steps: int, shift: float) -> TimestepSchedule:
        key = (round(denoise / DENOISE_QUANTUM), steps, shift)
        hit = self._entries.get(key)
        if hit is None:
            hit = self._entries[key] = build_schedule(denoise, steps, shift)
        return hit

    def __len__(self) -> int:
        return len(self._entries)


def migrate_schedule(current: TimestepSchedule, slot_step: int,
                     new: TimestepSchedule) -> TimestepSchedule:
    """Rebind a slot to ``new`` keeping its step index; only equal step counts."""
    if new.steps != current.steps:
        raise ScheduleMismatchError(
            f"cannot migrate across step counts ({current.steps} -> {new.steps})")
    if slot_step < 0 or slot_step > current.steps:
        raise ValueError(f"slot_step {slot_step} outside [0, {current.steps}]")
    return new
