"""The ring-buffer streaming pipeline: host bookkeeping + one batched device pass per tick.

Drop-in for reference ``pkg/src/ringflow/pipeline.py`` (``StreamPipeline`` :247-566 and
its types :56-244).  The split is the one SURVEY.md §8(a) prescribes:

* host (this file): slot table, submit queue, warmup pacing, schedule cache, shared
  registry, mode logic (per-slot / global-reset / migration), emit order, record
  bookkeeping -- all integer/id work, kept bit-identical to the reference;
* device (csrc/ via ctypes): every [T, D] byte -- keyed noise for all rows of the tick
  (one batched ``rf_normal_fill``), velocity + guidance + SDE/ODE update for all
  active rows (one ``rf_tick_solve``), emit statistics / copies (``rf_emit_stats``)
  and admissions (``rf_normal_fill`` + ``rf_admit_init``).

Ring state stays resident in HBM as float64 [depth, T, D]; the host reads back only
the per-emit statistics (mse vs last emitted, mse vs reference, non-finite flag) that
``CompletionRecord`` needs, so a tick with no completion does not synchronise.
All public methods serialise on one lock, as in the reference (pipeline.py:22-24):
a control write completed before tick N is visible to every step of tick N.
"""
from __future__ import annotations

import math
import threading
from collections import deque
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _device, _native
from ._native import RfAdmit, RfEmit, RfRow
from .latents import NoiseCache, NoiseSource, ShapeMismatchError, content_hash, fill_normals
from .model import UNCOND_PROMPT, ConditionSet, ModelWeights, ToyFlowModel
from .schedule import ScheduleCache, ScheduleMismatchError, TimestepSchedule, migrate_schedule
from .solver import (
    CURVE_FIELDS,
    CurveSet,
    MissingSourceError,
    StepState,
    clamp_curve,
    curve_pointers,
    guidance_plan,
    prepare_guidance_state,
)

__all__ = [
    "MODES",
    "BackpressureError",
    "GenerationRequest",
    "PipelineConfig",
    "CompletionRecord",
    "SharedRegistry",
    "SlotView",
    "PipelineSnapshot",
    "StreamPipeline",
    "StreamGroup",
]

MODES = ("per-slot", "global-reset", "migration")
_UNCOND = ConditionSet(prompt_hash=UNCOND_PROMPT)


class BackpressureError(RuntimeError):
    """The submit queue is at capacity; retry after a completion frees a slot."""


@dataclass(frozen=True)
class GenerationRequest:
    """Frozen per-generation request (pipeline.py:77-96)."""

    conditions: tuple
    curves: CurveSet = field(default_factory=CurveSet)
    solver: str = "sde"
    _cache: dict = field(default_factory=dict, init=False, repr=False, compare=False, hash=False)

    def __post_init__(self):
        if not self.conditions:
            raise ValueError("a request needs at least one condition")
        if self.solver not in ("sde", "ode"):
            raise ValueError("solver must be 'sde' or 'ode'")

    @property
    def source(self):
        return self.conditions[0].source

    def content_key(self) -> int:
        key = self._cache.get("key")
        if key is None:
            key = self._cache["key"] = content_hash([c.content_key() for c in self.conditions],
                                                    self.solver)
        return key


@dataclass(frozen=True)
class PipelineConfig:
    """Same fields and defaults as the reference (pipeline.py:99-128)."""

    depth: int = 8
    steps: int = 8
    frames: int = 96
    channels: int = 8
    frame_rate: float = 25.0
    mode: str = "per-slot"
    similarity_threshold: float = 1e-3
    seed: int = 0
    shift: float = 3.0
    denoise: float = 1.0
    model_jitter: float = 0.1
    auto_submit: bool = True

    def __post_init__(self):
        if self.depth < 1 or self.steps < 1:
            raise ValueError("depth and steps must be >= 1")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if not 0.0 < self.denoise <= 1.0:
            raise ValueError("denoise must be in (0, 1]")

    @property
    def shape(self):
        return (self.frames, self.channels)


class CompletionRecord:
    """One finished generation (pipeline.py:131-143).

    ``latent`` is materialised on the host on first access (the reference's numpy
    array); ``latent_device`` is the record-owned float64 copy in HBM.
    """

    __slots__ = ("latent_device", "tick", "completion_index", "submission_id", "schedule_id",
                 "denoise", "hybrid", "decode_skipped", "rms_vs_reference", "_host", "_stream")

    def __init__(self, latent_device, tick, completion_index, submission_id, schedule_id, denoise,
                 hybrid, decode_skipped, rms_vs_reference, stream=None):
        self.latent_device = latent_device
        self.tick = tick
        self.completion_index = completion_index
        self.submission_id = submission_id
        self.schedule_id = schedule_id
        self.denoise = denoise
        self.hybrid = hybrid
        self.decode_skipped = decode_skipped
        self.rms_vs_reference = rms_vs_reference
        self._host = None
        self._stream = stream

    @property
    def latent(self) -> np.ndarray:
        if self._host is None:
            if self._stream is not None:
                self._stream.synchronize()
            arr = self.latent_device.cpu().numpy()
            arr.setflags(write=False)
            self._host = arr
        return self._host

    def __repr__(self) -> str:
        return (f"CompletionRecord(tick={self.tick}, completion_index={self.completion_index}, "
                f"submission_id={self.submission_id}, schedule_id={self.schedule_id!r}, "
                f"denoise={self.denoise}, hybrid={self.hybrid}, decode_skipped={self.decode_skipped}, "
                f"rms_vs_reference={self.rms_vs_reference})")


class SharedRegistry:
    """Field-keyed hot-mutable per-step state (pipeline.py:146-184), mirrored in HBM.

    Every write replaces the field's device buffer, so work already enqueued keeps the
    value it was launched with and the next tick reads the new one.
    """

    def __init__(self, frames: int, channels: int):
        self._frames = frames
        self._channels = channels
        self._curves: dict = {}
        self._dev: dict = {}
        self._x0_target = None
        self._x0_dev = None
        self.write_count = 0

    def set(self, name: str, value) -> None:
        if name == "x0_target":
            if isinstance(value, torch.Tensor):
                host = value.detach().to("cpu", torch.float64).numpy()
            else:
                host = np.asarray(value, dtype=np.float64)
            if host.shape != (self._frames, self._channels):
                raise ValueError(f"x0_target must have shape {(self._frames, self._channels)}")
            self._x0_target = host
            self._x0_dev = _device.to_device_f64(host).clone()
        else:
            host = clamp_curve(name, value, self._frames)
            self._curves[name] = host
            self._dev[name] = _device.to_device_f64(host).clone()
        self.write_count += 1

    def overlay(self) -> dict:
        out = dict(self._curves)
        if self._x0_target is not None:
            out["x0_target"] = self._x0_target
        return out

    def device_overlay(self) -> dict:
        out = dict(self._dev)
        if self._x0_dev is not None:
            out["x0_target"] = self._x0_dev
        return out

    def digest(self) -> str:
        parts = [(name, self._curves[name]) for name in sorted(self._curves)]
        if self._x0_target is not None:
            parts.append(("x0_target", self._x0_target))
        return f"{self.write_count}:{content_hash(parts):016x}"


class _Slot:
    __slots__ = ("submission_id", "request", "denoise", "schedule", "x", "state", "rng",
                 "admitted_tick", "schedule_ids_used", "migrated", "_ring_index", "_row_tpl")

    def __init__(self, submission_id, request, denoise, schedule, x, state, rng, admitted_tick):
        self.submission_id = submission_id
        self.request = request
        self.denoise = denoise
        self.schedule = schedule
        self.x = x                      # device float64 [T, D] (a ring row)
        self.state = state
        self.rng = rng
        self.admitted_tick = admitted_tick
        self.schedule_ids_used = {schedule.schedule_id}
        self.migrated = False
        self._ring_index = None
        self._row_tpl = None            # (key, RfRow): the row's per-generation fields

    @property
    def step(self) -> int:
        return self.state.step


@dataclass(frozen=True)
class SlotView:
    denoise: float
    step: int
    schedule_id: str


@dataclass(frozen=True)
class PipelineSnapshot:
    slots: tuple
    queue_depth: int
    mode: str
    tick: int
    denoise: float

    def denoise_values(self) -> set:
        return {v.denoise for v in self.slots if v is not None}


@dataclass(frozen=True)
class _Submission:
    submission_id: int
    request: GenerationRequest
    denoise: float
    schedule: TimestepSchedule


class StreamPipeline:
    """submit() -> tick() -> CompletionRecord stream, computed on one CUDA stream."""

    def __init__(self, config: PipelineConfig, request: Optional[GenerationRequest] = None,
                 velocity_model=None, noise_cache_bytes: int = 256 << 20):
        """velocity_model: None (the reference's toy model, inside the fused solver) or a
        ``DiTVelocity``.  noise_cache_bytes: device budget of the keyed-noise cache
        (``NoiseCache``); 0 regenerates every draw every tick."""
        self.config = config
        self._dev = _device.device()
        self._stream = torch.cuda.Stream(self._dev)
        T, D = config.shape
        with torch.cuda.stream(self._stream):
            self.model = ToyFlowModel(T, D, perturbation=config.model_jitter)
            self.weights = ModelWeights.zeros(config.shape)
            self._ring = torch.zeros((config.depth, T, D), dtype=torch.float64, device=self._dev)
            # per slot: [0] model noise, [1] step noise (sde/ode), [2] admission noise
            self._noise = torch.empty((config.depth, 3, T, D), dtype=torch.float64, device=self._dev)
            # per-slot views made once (tensor indexing costs microseconds of host time per tick)
            self._noise_views = [[self._noise[i, j] for j in range(3)] for i in range(config.depth)]
            # emit statistics [2, depth] and the status word share one buffer (one read-back)
            nd = max(config.depth, 1)
            self._emitbuf = torch.zeros(2 * nd + 1, dtype=torch.float64, device=self._dev)
            self._stats = self._emitbuf[:2 * nd].view(2, nd)
            self._status = self._emitbuf[2 * nd:].view(torch.int32)[:1]
            self._stats_ptrs = (self._stats[0].data_ptr(), self._stats[1].data_ptr())
            # the emit reduction's partials: this pipeline's own (never shared across streams)
            self._reduce_elems = int(_native.load().rf_reduce_workspace_elems(T * D))
            # zeroed once: its tail holds rf_emit_stats' completion counters (left zero by every call)
            self._reduce_scratch = torch.zeros(max(self._reduce_elems, 1), dtype=torch.float64, device=self._dev)
        self.noise_cache = (NoiseCache(noise_cache_bytes, T * D, self._dev)
                            if noise_cache_bytes > 0 else None)
        self._emitbuf_host = torch.zeros(2 * nd + 1, dtype=torch.float64).pin_memory()
        self._stats_host = self._emitbuf_host[:2 * nd].view(2, nd)
        self._status_host = self._emitbuf_host[2 * nd:].view(torch.int32)[:1]
        self._emit_event = torch.cuda.Event()
        self.velocity_model = velocity_model   # None: the toy model inside the fused kernel
        self.cache = ScheduleCache()
        self.registry = SharedRegistry(T, D)
        self.mode = config.mode
        self.denoise = config.denoise
        self._template = request
        self._slots: list = [None] * config.depth
        self._queue: deque = deque()
        self._lock = threading.RLock()
        self._tick_index = 0
        self._completions = 0
        self._submissions = 0
        self._prev_tick_denoise = config.denoise
        self._reference = None            # device tensor
        self._last_emitted = None         # device tensor
        self._spacing = math.ceil(config.steps / config.depth)
        self._warmup_left = config.depth
        self._last_admit: Optional[int] = None
        self.migration_refusals = 0
        self.last_timesteps: list = []
        self.launches_last_tick = 0
        self.rows_last_tick = 0
        self._phases = None  # {phase: [(start_event, end_event), ...]} when timing is on
        self._last_solve = None
        self._views: dict = {}            # id(request) -> cached curve view (see _curve_view)
        self._views_version = -1

    # ------------------------------------------------------------- profiling
    def enable_phase_timing(self, on: bool = True) -> dict:
        """Record CUDA events (on this pipeline's stream) around each device phase."""
        self._phases = {} if on else None
        return self._phases

    def _phase_begin(self, name):
        if self._phases is None:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self._stream)
        return ev

    def _phase_end(self, name, start):
        if start is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self._stream)
        self._phases.setdefault(name, []).append((start, ev))

    # ------------------------------------------------------------------ state
    @property
    def tick_index(self) -> int:
        return self._tick_index

    @property
    def completions_total(self) -> int:
        return self._completions

    @property
    def queue_depth(self) -> int:
        return len(self._queue)

    @property
    def stream(self) -> torch.cuda.Stream:
        return self._stream

    def snapshot(self) -> PipelineSnapshot:
        with self._lock:
            views = tuple(None if s is None else SlotView(s.denoise, s.step, s.schedule.schedule_id)
                          for s in self._slots)
            return PipelineSnapshot(views, len(self._queue), self.mode, self._tick_index, self.denoise)

    # ---------------------------------------------------------------- control
    def _mark_reference(self) -> None:
        if self._last_emitted is not None:
            self._reference = self._last_emitted  # records are immutable: no copy needed

    def set_request(self, request: GenerationRequest) -> int:
        with self._lock:
            self._mark_reference()
            self._template = request
            return self._tick_index

    def set_denoise(self, value: float) -> int:
        if not 0.0 < value <= 1.0:
            raise ValueError("denoise must be in (0, 1]")
        with self._lock:
            self._mark_reference()
            self.denoise = float(value)
            return self._tick_index

    def set_shared_curve(self, name: str, value) -> int:
        with self._lock, _device.on_stream(self._stream):
            self._mark_reference()
            self.registry.set(name, value)
            return self._tick_index

    def set_model_weights(self, offset) -> int:
        with self._lock, _device.on_stream(self._stream):
            self._mark_reference()
            self.weights.swap_offset(offset)
            return self._tick_index

    def set_mode(self, mode: str) -> int:
        if mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        with self._lock:
            self._mark_reference()
            self.mode = mode
            self._prev_tick_denoise = self.denoise
            return self._tick_index

    # ----------------------------------------------------------------- submit
    def submit(self, request: Optional[GenerationRequest] = None) -> int:
        with self._lock:
            if len(self._queue) >= self.config.depth:
                raise BackpressureError(f"submit queue at capacity ({self.config.depth})")
            return self._enqueue(request)

    def _enqueue(self, request: Optional[GenerationRequest]) -> int:
        request = request if request is not None else self._template
        if request is None:
            raise ValueError("no request given and no template set")
        if self.denoise < 1.0 and request.source is None:
            raise ValueError("denoise < 1 requires source latents in the request")
        sub = _Submission(self._submissions, request, self.denoise,
                          self.cache.get(self.denoise, self.config.steps, self.config.shift))
        self._submissions += 1
        self._queue.append(sub)
        return sub.submission_id

    # ------------------------------------------------------------- validation
    def _check_request(self, request: GenerationRequest) -> None:
        """Host-side checks the reference makes inside the step (every pointer the kernels
        dereference must cover [T, D] / [T]): a source of the wrong shape raises
        ShapeMismatchError as ``sde_step`` does (solver.py:300-301), a weight curve of the
        wrong shape, a negative weight or a zero weight sum raises ValueError as
        ``blend_conditions`` does (solver.py:217-226).  Checked once per (request, shape):
        requests are frozen and their arrays are read-only copies (model.py)."""
        shape = self.config.shape
        key = ("checked", shape)
        if request._cache.get(key):  # noqa: SLF001
            return
        for c in request.conditions:
            if c.source is not None and tuple(c.source.shape) != shape:
                raise ShapeMismatchError(f"source shape {tuple(c.source.shape)} != {shape}")
        if len(request.conditions) > 1:
            total = np.zeros(shape[0])
            for c in request.conditions:
                w = np.ones(shape[0]) if c.weight_curve is None else c.weight_curve
                if tuple(w.shape) != (shape[0],):
                    raise ValueError(f"weight_curve shape {tuple(w.shape)} != ({shape[0]},)")
                if np.any(w < 0.0):
                    raise ValueError("condition weights must be nonnegative")
                total = total + w
            if np.any(total <= 0.0):
                raise ValueError("condition weights sum to zero at some frame")
        curves = request.curves
        for name in CURVE_FIELDS:
            val = getattr(curves, name)
            if val is not None and tuple(val.shape) != (shape[0],):
                raise ShapeMismatchError(f"{name} must have shape ({shape[0]},), got {tuple(val.shape)}")
        if curves.x0_target is not None and tuple(np.shape(curves.x0_target)) != shape:
            raise ShapeMismatchError(f"x0_target shape {tuple(np.shape(curves.x0_target))} != {shape}")
        request._cache[key] = True  # noqa: SLF001

    # ------------------------------------------------------------------- tick
    def tick(self) -> list:
        """Advance every in-flight slot one step; emit finished latents (pipeline.py:372-398)."""
        with self._lock, _device.on_stream(self._stream):
            active = self._tick_begin()
            if active:
                self._step_slots(active)
            return self._tick_end()

    def _tick_begin(self) -> list:
        """Mode pre-pass and the active slots of this tick (pipeline.py:372-385)."""
        self.launches_last_tick = 0
        if self.mode == "migration":
            self._migration_pass()
        if self.mode == "global-reset" and self.denoise != self._prev_tick_denoise:
            self._slots = [None] * self.config.depth
            self._warmup_left = self.config.depth
            self._last_admit = None
        active = [s for s in self._slots if s is not None]
        self.last_timesteps = [(s.schedule.sigmas[s.step], s.schedule.schedule_id) for s in active]
        return active

    def _tick_end(self) -> list:
        """Emit finished slots, refill, advance the tick counter (pipeline.py:386-398)."""
        finished = [(i, s) for i, s in enumerate(self._slots) if s is not None and s.step >= self.config.steps]
        # emit: the statistics kernel and its read-back are queued, the finished slots are
        # refilled (admission kernels queued behind them), and only then does the host wait
        # for the device to build the records
        pending = self._emit_launch(finished) if finished else None
        for i, _ in finished:
            self._slots[i] = None
        self._refill()
        records = self._emit_finish(finished, *pending) if finished else []
        self._prev_tick_denoise = self.denoise
        self._tick_index += 1
        return records

    def _migration_pass(self) -> None:
        target = self.cache.get(self.denoise, self.config.steps, self.config.shift)
        for slot in self._slots:
            if slot is None or slot.schedule.schedule_id == target.schedule_id:
                continue
            try:
                slot.schedule = migrate_schedule(slot.schedule, slot.step, target)
            except ScheduleMismatchError:
                self.migration_refusals += 1
                continue
            slot.denoise = target.denoise
            slot.schedule_ids_used.add(target.schedule_id)
            slot.migrated = True

    def _curve_view(self, slot: _Slot):
        """Effective curves of a slot this step (pipeline.py:415-422): (host dict, device
        dict, the request's CurveSet, the solver's curve-pointer array).  A view depends
        only on the request and the registry's contents, so it is built once per (request,
        registry write) and reused by every slot and tick until the next registry write."""
        req = slot.request
        version = self.registry.write_count
        if self._views_version != version:
            self._views.clear()
            self._views_version = version
        view = self._views.get(id(req))
        if view is None or view[0] is not req:
            host, dev, base = self._build_curve_view(slot)
            ptrs = (_native.c_dptr * _native.RF_NUM_CURVES)()
            for name, idx in _native.CURVE_INDEX.items():
                t = dev[name]
                ptrs[idx] = None if t is None else t.data_ptr()
            view = (req, host, dev, base, ptrs)
            self._views[id(req)] = view
        return view[1], view[2], view[3], view[4]

    def _build_curve_view(self, slot: _Slot):
        base = slot.request.curves
        reg_host = self.registry.overlay()
        reg_dev = self.registry.device_overlay()
        host, dev = {}, {}
        for name in CURVE_FIELDS:
            if name in reg_host:
                host[name], dev[name] = reg_host[name], reg_dev[name]
            else:
                host[name], dev[name] = getattr(base, name), base.device(name)
        if "x0_target" in reg_host:
            host["x0_target"], dev["x0_target"] = reg_host["x0_target"], reg_dev["x0_target"]
        else:
            host["x0_target"], dev["x0_target"] = base.x0_target, base.device("x0_target")
        if host["x0_target"] is None:
            host["x0_target_strength"] = dev["x0_target_strength"] = None
        return host, dev, base

    def _model_rows(self, slots: list) -> list:
        """The velocity model's rows of this tick (one per slot x condition, + uncond rows),
        queued on the model; returns the solver row descriptors they feed."""
        rows = [RfRow() for _ in slots]
        try:
            for slot, row in zip(slots, rows):
                base = slot.request.curves
                need_uncond = (base.guidance_enabled and
                               guidance_plan(base.rcfg_mode, slot.state, True)[0] == _native.RF_NEG_UNCOND)
                self.velocity_model.prepare_row(self, slot, row, float(slot.schedule.sigmas[slot.step]),
                                                need_uncond)
        except BaseException:
            self.velocity_model.reset()
            raise
        return rows

    def _step_slots(self, slots: list, rows: Optional[list] = None) -> None:
        """One batched pass over `slots`: noise for every row, then one fused solve.
        rows: model rows already prepared and forwarded by a ``StreamGroup``."""
        cfg = self.config
        for slot in slots:
            self._check_request(slot.request)
        T, D = cfg.shape
        jitter = self.model.perturbation
        draws = []
        if self.velocity_model is not None and rows is None:
            # the DiT's inputs first: its (long) batched forward is launched before the host
            # prepares the solver rows, so that host work overlaps the device work
            rows = self._model_rows(slots)
            ev = self._phase_begin("model")
            self.velocity_model.forward(self)
            self._phase_end("model", ev)
            self.launches_last_tick += getattr(self.velocity_model, "launches_per_forward", 0)
        elif rows is None:
            rows = []
        for i, slot in enumerate(slots):
            k = slot.step
            t_curr = float(slot.schedule.sigmas[k])
            t_next = float(slot.schedule.sigmas[k + 1])
            host, dev, base, curve_ptrs = self._curve_view(slot)
            req = slot.request
            nbuf = self._noise_buffers(slot)
            if self.velocity_model is None:
                row = _native.RfRow.from_buffer_copy(self._row_template(slot, host, base, curve_ptrs))
                if jitter != 0.0:
                    row.noise_model = self._noise_for(slot.rng.key(k, "model"), nbuf[0], draws).data_ptr()
                    row.jitter_t = jitter * t_curr
            else:
                row = rows[i]
                self._row_static(row, slot, host, base, curve_ptrs)
            row.t_curr, row.t_next = t_curr, t_next
            if base.guidance_enabled:
                neg_kind, flags = guidance_plan(base.rcfg_mode, slot.state, True)
                row.neg_kind, row.flags = neg_kind, row.flags | flags
                prepare_guidance_state(row, slot.state, host["apg_momentum"] is not None, slot.x)
            refine = host["x0_target"] is not None and slot.state.in_refinement_half()
            if req.solver == "sde":
                row.noise_step = self._noise_for(slot.rng.key(k, "sde"), nbuf[1], draws).data_ptr()
                if refine:
                    row.x0_target = dev["x0_target"].data_ptr()
            else:
                if refine:
                    row.flags |= _native.RF_ROWF_ODE_MORPH
                    row.x0_target = dev["x0_target"].data_ptr()
                if host["ode_noise_curve"] is not None:
                    row.noise_step = self._noise_for(slot.rng.key(k, "ode"), nbuf[1], draws).data_ptr()
            if self.velocity_model is None:
                rows.append(row)
        if draws:
            ev = self._phase_begin("noise")
            fill_normals(draws, self._status, self._stream.cuda_stream)
            if self.noise_cache is not None:
                self.noise_cache.filled(key for key, _ in draws)
            self._phase_end("noise", ev)
            self.launches_last_tick += 2
        lib = _native.load()
        arr = (RfRow * len(rows))(*rows)
        self._last_solve = (arr, len(rows))   # kept for bench.py's per-launch solver timing
        ev = self._phase_begin("solve")
        _native.check(lib.rf_tick_solve(arr, len(rows), T, D, self.weights.device_offset.data_ptr(),
                                        self._stream.cuda_stream), "rf_tick_solve")
        if self.velocity_model is not None:
            self.velocity_model.consumed(self._stream)
        self._phase_end("solve", ev)
        self.launches_last_tick += 1
        self.rows_last_tick = len(rows)
        for slot in slots:
            slot.state.step += 1
            slot.schedule_ids_used.add(slot.schedule.schedule_id)

    def _noise_for(self, key: int, fallback: torch.Tensor, draws: list) -> torch.Tensor:
        """The device draw for ``key``: a noise-cache entry (queued for generation on a
        miss) or, without the cache, ``fallback`` (always queued)."""
        if self.noise_cache is None:
            draws.append((key, fallback))
            return fallback
        buf, hit = self.noise_cache.lookup(key, self._tick_index)
        if not hit:
            draws.append((key, buf))
        return buf

    def _row_static(self, row, slot: _Slot, host: dict, base, curve_ptrs) -> None:
        """Row fields fixed for a slot's generation (until a registry / weights write):
        latent, conditions, curves, solver and source (reference pipeline.py:424-464)."""
        req = slot.request
        row.x = slot.x.data_ptr()
        if self.velocity_model is None:
            conds = req.conditions
            row.n_cond = len(conds)
            if row.n_cond > _native.RF_MAX_COND:
                raise NotImplementedError(f"at most {_native.RF_MAX_COND} conditions per request")
            for j, c in enumerate(conds):
                row.cond_x0[j] = self.model.x0_partial(c).data_ptr()
                if len(conds) > 1:
                    w = c.weight_device()
                    row.cond_w[j] = None if w is None else w.data_ptr()
            if base.guidance_enabled:
                row.uncond_x0 = self.model.x0_partial(_UNCOND).data_ptr()
        elif self.weights.version > 0:
            row.flags |= _native.RF_ROWF_STYLE_V   # set_model_weights on the DiT path
        row.curves = curve_ptrs
        if req.solver == "sde":
            src = req.conditions[0].source_device()
            if src is None:
                curve = host["sde_denoise_curve"]
                if curve is not None and np.any(curve < 1.0):
                    raise MissingSourceError("sde_denoise_curve < 1 requires source latents")
            row.solver = _native.RF_SOLVER_SDE
            row.source = None if src is None else src.data_ptr()
        else:
            row.solver = _native.RF_SOLVER_ODE

    def _row_template(self, slot: _Slot, host: dict, base, curve_ptrs):
        """The toy-path row's static fields, built once per (slot, registry write, weights
        write) and copied per tick."""
        key = (self._views_version, self.weights.version)
        tpl = slot._row_tpl  # noqa: SLF001
        if tpl is None or tpl[0] != key:
            row = _native.RfRow()
            self._row_static(row, slot, host, base, curve_ptrs)
            tpl = slot._row_tpl = (key, row)  # noqa: SLF001
        return tpl[1]

    def _noise_buffers(self, slot: _Slot):
        idx = slot._ring_index  # noqa: SLF001
        if idx is None:  # render(): private buffers
            return list(slot.x.new_empty((3,) + tuple(slot.x.shape)))
        return self._noise_views[idx]

    def _emit(self, finished: list) -> list:
        """_emit for every finished slot, in slot-index order (pipeline.py:466-491)."""
        return self._emit_finish(finished, *self._emit_launch(finished))

    def _emit_launch(self, finished: list):
        """Queue the emit statistics (isfinite, mse vs the last emitted / the reference)."""
        cfg = self.config
        n = len(finished)
        for _, slot in finished:
            if len(slot.schedule_ids_used) > 1 and not slot.migrated:
                raise RuntimeError("single-schedule trajectory invariant violated")
        recs_dev = [torch.empty_like(slot.x) for _, slot in finished]
        emits = (RfEmit * n)()
        for j, (_, slot) in enumerate(finished):
            emits[j].latent = slot.x.data_ptr()
            emits[j].record = recs_dev[j].data_ptr()
        lib = _native.load()
        last = self._last_emitted
        ref = self._reference
        ev = self._phase_begin("emit")
        _native.check(lib.rf_emit_stats(
            emits, n, slot.x.numel(), None if last is None else last.data_ptr(),
            None if ref is None else ref.data_ptr(), self._stats_ptrs[0],
            self._stats_ptrs[1], self._status.data_ptr(), self._reduce_scratch.data_ptr(),
            self._reduce_elems, self._stream.cuda_stream),
            "rf_emit_stats")
        self._phase_end("emit", ev)
        self.launches_last_tick += 1
        self._emitbuf_host.copy_(self._emitbuf, non_blocking=True)
        done = self._emit_event
        done.record(self._stream)
        return recs_dev, done

    def _emit_finish(self, finished: list, recs_dev: list, done) -> list:
        """Wait for the statistics and build the CompletionRecords (pipeline.py:466-491)."""
        cfg = self.config
        done.synchronize()
        status = int(self._status_host[0])
        if status & _native.RF_STATUS_NONFINITE:
            raise RuntimeError("non-finite completion latent; aborting session")
        if status & _native.RF_STATUS_NOISE_SHORT:
            raise RuntimeError("keyed noise generation ran out of stream positions")
        stats = self._stats_host.numpy()
        records = []
        for j, (_, slot) in enumerate(finished):
            has_prev = j > 0 or self._last_emitted is not None
            skipped = bool(has_prev and stats[0, j] < cfg.similarity_threshold)
            rms = float(np.sqrt(stats[1, j])) if self._reference is not None else None
            rec = CompletionRecord(recs_dev[j], self._tick_index, self._completions, slot.submission_id,
                                   slot.schedule.schedule_id, slot.denoise,
                                   len(slot.schedule_ids_used) > 1, skipped, rms, self._stream)
            self._completions += 1
            self._last_emitted = recs_dev[j]
            records.append(rec)
        return records

    # ----------------------------------------------------------------- refill
    def _admission_allowed(self) -> bool:
        if self._warmup_left <= 0 or self._last_admit is None:
            return True
        return self._tick_index - self._last_admit >= self._spacing

    def _refill(self) -> None:
        """End-of-tick refill with warmup pacing (pipeline.py:502-521)."""
        admitted = []
        try:
            for idx in range(self.config.depth):
                if self._slots[idx] is not None:
                    continue
                if not self._admission_allowed():
                    break
                if self._queue:
                    sub = self._queue.popleft()
                elif self.config.auto_submit and self._template is not None:
                    self._enqueue(None)
                    sub = self._queue.popleft()
                else:
                    break
                slot = self._new_slot(sub, self._ring[idx])
                slot._ring_index = idx  # noqa: SLF001 - slots carry their ring row
                self._slots[idx] = slot
                admitted.append(slot)
                if self._warmup_left > 0:
                    self._warmup_left -= 1
                self._last_admit = self._tick_index
        finally:
            if admitted:
                self._init_slots(admitted)

    def _new_slot(self, sub: _Submission, x: torch.Tensor) -> _Slot:
        if sub.denoise < 1.0 and sub.request.source is None:
            raise RuntimeError("denoise < 1 admission without source")
        rng = NoiseSource(seed=self.config.seed, stream=sub.request.content_key())
        return _Slot(sub.submission_id, sub.request, sub.denoise, sub.schedule, x,
                     StepState(steps_total=self.config.steps), rng, self._tick_index)

    def _init_slots(self, slots: list) -> None:
        """Admission draws + x = n or d*n + (1-d)*source for all new slots (pipeline.py:523-532)."""
        for slot in slots:
            self._check_request(slot.request)
        draws, admits = [], (RfAdmit * len(slots))()
        for j, slot in enumerate(slots):
            nbuf = self._noise_for(slot.rng.key(0, "init"), self._noise_buffers(slot)[2], draws)
            admits[j].x = slot.x.data_ptr()
            admits[j].noise = nbuf.data_ptr()
            if slot.denoise < 1.0:
                admits[j].source = slot.request.conditions[0].source_device().data_ptr()
                admits[j].denoise = slot.denoise
            else:
                admits[j].source = None
                admits[j].denoise = 1.0
        ev = self._phase_begin("admit")
        if draws:
            fill_normals(draws, self._status, self._stream.cuda_stream)
            if self.noise_cache is not None:
                self.noise_cache.filled(key for key, _ in draws)
        lib = _native.load()
        _native.check(lib.rf_admit_init(admits, len(slots), slots[0].x.numel(), self._stream.cuda_stream),
                      "rf_admit_init")
        self._phase_end("admit", ev)
        self.launches_last_tick += 3 if draws else 1

    # ----------------------------------------------------- sequential renderer
    def render(self, request: Optional[GenerationRequest] = None, denoise: Optional[float] = None):
        """Batch-mode oracle through the same step code (pipeline.py:546-566)."""
        with self._lock, _device.on_stream(self._stream):
            request = request if request is not None else self._template
            if request is None:
                raise ValueError("no request given and no template set")
            d = self.denoise if denoise is None else denoise
            schedule = self.cache.get(d, self.config.steps, self.config.shift)
            x = torch.empty(self.config.shape, dtype=torch.float64, device=self._dev)
            slot = self._new_slot(_Submission(-1, request, d, schedule), x)
            self._init_slots([slot])
            for _ in range(self.config.steps):
                self._step_slots([slot])
            out = x.cpu().numpy()
            return out


class StreamGroup:
    """Co-resident streams on one GPU ticked together with ONE batched DiT forward
    ("rows of several co-resident streams may be batched into one DiT
    forward").  Every pipeline keeps its own ring, registry, schedules and CUDA stream;
    per tick the group gathers every pipeline's model rows (their slots x conditions, +
    unconditional rows), runs one forward on the group's stream, then each pipeline solves,
    emits and refills on its own stream.  DiT rows are independent (no cross-row reduction
    in any kernel), so each stream's completions are bit-identical to ticking it alone.

    All pipelines must share ``velocity_model`` (one ``DiTVelocity`` whose DiT has
    ``max_rows`` >= the rows of all streams together)."""

    def __init__(self, pipelines: list):
        if not pipelines:
            raise ValueError("a stream group needs at least one pipeline")
        vm = pipelines[0].velocity_model
        if vm is None or any(p.velocity_model is not vm for p in pipelines):
            raise ValueError("the pipelines of a group must share one DiT velocity model")
        self.pipelines = list(pipelines)
        self.velocity_model = vm
        self._stream = torch.cuda.Stream(pipelines[0]._dev)  # noqa: SLF001

    @property
    def stream(self) -> torch.cuda.Stream:
        return self._stream

    def tick(self) -> list:
        """One tick of every stream; returns one list of CompletionRecords per pipeline."""
        pipes = self.pipelines
        for p in pipes:
            p._lock.acquire()  # noqa: SLF001
        try:
            begun = []
            for p in pipes:
                with torch.cuda.stream(p.stream):
                    active = p._tick_begin()  # noqa: SLF001
                    rows = p._model_rows(active) if active else []  # noqa: SLF001
                begun.append((active, rows))
            if any(a for a, _ in begun):
                for p in pipes:   # the forward reads every ring's latents as of its last step
                    self._stream.wait_stream(p.stream)
                with torch.cuda.stream(self._stream):
                    self.velocity_model.forward(None)
                done = torch.cuda.Event()
                done.record(self._stream)
            out, counted = [], False
            for p, (active, rows) in zip(pipes, begun):
                with torch.cuda.stream(p.stream):
                    if active:
                        p.stream.wait_event(done)
                        if not counted:   # the shared forward's kernels, counted once
                            p.launches_last_tick += getattr(self.velocity_model, "launches_per_forward", 0)
                            counted = True
                        p._step_slots(active, rows)  # noqa: SLF001
                    out.append(p._tick_end())  # noqa: SLF001
            return out
        finally:
            for p in pipes:
                p._lock.release()  # noqa: SLF001
