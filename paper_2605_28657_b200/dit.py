"""ACE-Step-1.5-shape DiT velocity model (BASELINE configs 2-5) on sm_100a kernels.

The reference package has no DiT (its ``ToyFlowModel`` is a closed-form stand-in,
reference model.py:91-152).  The paper's production model is ACE-Step 1.5
(24-layer DiT, AdaLN, RMSNorm, GQA attention + MLP, 64-channel latent at 25 Hz;
PAPER.md:44,226,242).  This module defines a builder-chosen model of that shape
(``DiTConfig`` defaults; DESIGN.md lists every choice) with seeded random weights:

    patch 2 (T=1500 frames -> 750 tokens), d=2048, 24 layers, 16 query / 8 KV heads of
    128, SwiGLU 6144, RMSNorm, AdaLN-single timestep modulation, RoPE, cross-attention
    to 128 conditioning tokens per prompt, fp32 residual stream.

The forward is one C-ABI call (``rf_dit_forward``, csrc/rf_dit.cu): tcgen05 GEMMs fed by
TMA with fused epilogues (RoPE, SwiGLU, AdaLN-gated residual), flash attention, fused
RMSNorm+modulation.  ``oracle/dit_fp32.py`` is the same network in plain PyTorch fp32 --
the oracle the DiT is tested against (DiT parity is unpinned by the reference itself).
"""
from __future__ import annotations

import ctypes
import threading
import math
from dataclasses import dataclass, field

import torch

from . import _device, _native


class RfDitConfig(ctypes.Structure):
    _fields_ = [("latent_channels", ctypes.c_int32), ("patch", ctypes.c_int32), ("d_model", ctypes.c_int32),
                ("n_layers", ctypes.c_int32), ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("mlp_hidden", ctypes.c_int32), ("n_cond_tokens", ctypes.c_int32),
                ("freq_dim", ctypes.c_int32), ("rope_theta", ctypes.c_float), ("norm_eps", ctypes.c_float)]


_WNAMES = ("w_in", "w_t1", "w_t2", "w_ada", "ada_table", "w_qkv", "w_o", "w_qc", "w_kvc", "w_oc", "w_gu", "w_down",
           "w_final_ada", "w_out", "ones")


class RfDitWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in _WNAMES]


def _declare(lib):
    if getattr(lib, "_dit_declared", False):
        return
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.rf_dit_workspace_bytes.restype = i64
    lib.rf_dit_workspace_bytes.argtypes = [ctypes.POINTER(RfDitConfig), i32, i32]
    lib.rf_dit_create.restype = ctypes.c_int
    lib.rf_dit_create.argtypes = [ctypes.POINTER(RfDitConfig), ctypes.POINTER(RfDitWeights), i32, i32, vp, i64,
                                  ctypes.POINTER(vp), vp]
    lib.rf_dit_destroy.restype = ctypes.c_int
    lib.rf_dit_destroy.argtypes = [vp]
    lib.rf_dit_launches.restype = ctypes.c_int
    lib.rf_dit_launches.argtypes = [vp, i32]
    lib.rf_dit_forward.restype = ctypes.c_int
    lib.rf_dit_forward.argtypes = [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_float), ctypes.POINTER(vp),
                                   vp, vp]
    lib.rf_dit_output.restype = vp
    lib.rf_dit_output.argtypes = [vp]
    lib.rf_attention_tc_bf16.restype = ctypes.c_int
    lib.rf_attention_tc_bf16.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i64, i64, i64, vp]
    lib._dit_declared = True


@dataclass(frozen=True)
class DiTConfig:
    latent_channels: int = 64
    patch: int = 2
    d_model: int = 2048
    n_layers: int = 24
    n_heads: int = 16
    n_kv_heads: int = 8
    head_dim: int = 128
    mlp_hidden: int = 6144
    n_cond_tokens: int = 128
    freq_dim: int = 256
    rope_theta: float = 10000.0
    norm_eps: float = 1e-6
    seed: int = 1234

    @property
    def in_dim(self):
        return self.patch * self.latent_channels

    def params(self) -> int:
        d, L = self.d_model, self.n_layers
        q, kv = self.n_heads * self.head_dim, self.n_kv_heads * self.head_dim
        per_layer = d * (q + 2 * kv) + q * d + d * q + d * 2 * kv + q * d + 3 * d * self.mlp_hidden
        return L * per_layer + d * self.in_dim * 2 + d * self.freq_dim + d * d + 8 * d * d

    def flops_per_forward(self, rows: int, frames: int) -> float:
        """Algorithmic FLOPs of one batched forward (GEMMs + attention matmuls)."""
        N = frames // self.patch
        d, L, F = self.d_model, self.n_layers, self.mlp_hidden
        q, kv, Nc = self.n_heads * self.head_dim, self.n_kv_heads * self.head_dim, self.n_cond_tokens
        tok = 2 * (d * (q + 2 * kv) + q * d + d * q + q * d + d * 2 * F + F * d)
        per_row = L * (N * tok + 2 * Nc * d * 2 * kv + 4 * N * N * q + 4 * N * Nc * q)
        per_row += 2 * N * self.in_dim * d * 2
        return float(rows) * per_row

    def small(self, **kw) -> "DiTConfig":
        base = dict(self.__dict__)
        base.update(dict(d_model=256, n_layers=2, n_heads=2, n_kv_heads=1, mlp_hidden=512, n_cond_tokens=32))
        base.update(kw)
        return DiTConfig(**base)

    def to_c(self) -> RfDitConfig:
        return RfDitConfig(self.latent_channels, self.patch, self.d_model, self.n_layers, self.n_heads,
                           self.n_kv_heads, self.head_dim, self.mlp_hidden, self.n_cond_tokens, self.freq_dim,
                           self.rope_theta, self.norm_eps)


class DiTWeights:
    """Seeded random-init weights (bf16 [out, in] matrices, fp32 tables) resident in HBM."""

    def __init__(self, cfg: DiTConfig, device=None):
        dev = device or _device.device()
        g = torch.Generator(device=dev).manual_seed(cfg.seed)
        d, L, F = cfg.d_model, cfg.n_layers, cfg.mlp_hidden
        q, kv = cfg.n_heads * cfg.head_dim, cfg.n_kv_heads * cfg.head_dim

        def lin(*shape, std=None):
            fan_in = shape[-1]
            s = std if std is not None else 1.0 / math.sqrt(fan_in)
            return (torch.randn(*shape, generator=g, device=dev) * s).to(torch.bfloat16).contiguous()

        self.w_in = lin(d, cfg.in_dim)
        self.w_t1 = lin(d, cfg.freq_dim)
        self.w_t2 = lin(d, d)
        self.w_ada = lin(6 * d, d, std=0.02)
        self.ada_table = (torch.randn(L, 6 * d, generator=g, device=dev) * 0.1).contiguous()
        self.w_qkv = lin(L, q + 2 * kv, d)
        self.w_o = lin(L, d, q)
        self.w_qc = lin(L, q, d)
        self.w_kvc = lin(L, 2 * kv, d)
        self.w_oc = lin(L, d, q)
        gate, up = lin(L, F, d), lin(L, F, d)
        self.w_gu = torch.stack([gate, up], dim=2).reshape(L, 2 * F, d).contiguous()  # rows (g_j, u_j)
        self.w_down = lin(L, d, F)
        self.w_final_ada = lin(2 * d, d, std=0.02)
        self.w_out = lin(cfg.in_dim, d)
        self.ones = torch.ones(d, device=dev, dtype=torch.float32)

    def to_c(self) -> RfDitWeights:
        return RfDitWeights(*[getattr(self, n).data_ptr() for n in _WNAMES])


class DiT:
    """Batched DiT forward over ring rows, each with its own timestep and conditioning."""

    def __init__(self, cfg: DiTConfig = DiTConfig(), frames: int = 1500, max_rows: int = 8, weights=None):
        self.cfg = cfg
        self.frames = frames
        self.max_rows = max_rows
        self.dev = _device.device()
        self.lib = _native.load()
        _declare(self.lib)
        self.weights = weights or DiTWeights(cfg, self.dev)
        self._ccfg = cfg.to_c()
        self._cw = self.weights.to_c()
        nbytes = self.lib.rf_dit_workspace_bytes(ctypes.byref(self._ccfg), max_rows, frames)
        if nbytes < 0:
            raise _native.NativeError("rf_dit_workspace_bytes failed")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        h = ctypes.c_void_p()
        _native.check(self.lib.rf_dit_create(ctypes.byref(self._ccfg), ctypes.byref(self._cw), max_rows, frames,
                                             self.workspace.data_ptr(), nbytes, ctypes.byref(h),
                                             _device.current_stream_handle()), "rf_dit_create")
        self.handle = h
        self._cond: dict = {}
        self.out = torch.empty(max_rows, frames, cfg.latent_channels, dtype=torch.float32, device=self.dev)
        # The handle's workspace, row table, captured graphs and ``out`` are shared mutable
        # device state: a forward on one stream must not start while earlier work using them
        # (a forward, or a solver reading the velocities) on another stream is in flight.
        # One event per stream that used them; the allocator is told about every such
        # stream (record_stream), so their memory is not reused before that work is done.
        self._busy: dict = {}
        # host-side state of the handle (row table, captured graphs per row count) is built
        # and replayed by one thread at a time
        self._lock = threading.Lock()
        # weights, tables and the handle were initialised on the creating stream: complete
        # them before any other stream can touch them
        torch.cuda.current_stream(self.dev).synchronize()

    def mark_used(self, stream=None) -> None:
        """Record that work reading this DiT's buffers was queued on ``stream`` (default:
        current); the next forward on a different stream waits for it."""
        stream = stream or torch.cuda.current_stream(self.dev)
        ev = self._busy.get(stream)
        if ev is None:
            self.workspace.record_stream(stream)
            self.out.record_stream(stream)
            ev = self._busy[stream] = torch.cuda.Event()
        ev.record(stream)

    def _order_after_previous_use(self) -> None:
        cur = torch.cuda.current_stream(self.dev)
        for stream, ev in self._busy.items():
            if stream != cur:
                cur.wait_event(ev)

    def __del__(self):
        try:
            for ev in getattr(self, "_busy", {}).values():
                ev.synchronize()   # in-flight graph replays still use the handle's buffers
            if getattr(self, "handle", None):
                self.lib.rf_dit_destroy(self.handle)
        except Exception:
            pass

    def _tokens(self, prompt_hash: int, kind: str) -> torch.Tensor:
        key = (prompt_hash, kind)
        t = self._cond.get(key)
        if t is None:
            salt = {"base": 0, "hint": 0x5A17, "timbre": 0x7B1E}[kind]
            g = torch.Generator(device=self.dev).manual_seed((int(prompt_hash) ^ salt) & ((1 << 62) - 1))
            t = torch.randn(self.cfg.n_cond_tokens, self.cfg.d_model, generator=g, device=self.dev)
            self._cond[key] = t
        return t

    def cond_tokens(self, prompt_hash: int, hint: float = 0.0, timbre: float = 0.0) -> torch.Tensor:
        """Conditioning tokens of a condition: a seeded stand-in for the text / lyric encoder
        output, plus the audio-hint and timbre embeddings scaled by the condition's
        strengths (the DiT-side reading of model.py:123-131's
        x0 = base + 0.45 h hint + 0.45 tau timbre).  Composed once per condition and cached."""
        key = ("cond", prompt_hash, float(hint), float(timbre))
        t = self._cond.get(key)
        if t is None:
            t = self._tokens(prompt_hash, "base")
            if hint != 0.0:
                t = t + (0.45 * hint) * self._tokens(prompt_hash, "hint")
            if timbre != 0.0:
                t = t + (0.45 * timbre) * self._tokens(prompt_hash, "timbre")
            t = t.to(torch.bfloat16).contiguous()
            # cached tokens are read from any stream (every pipeline sharing this DiT):
            # finish creating them before handing them out
            torch.cuda.current_stream(self.dev).synchronize()
            self._cond[key] = t
        return t

    def forward(self, xs, ts, conds, out: torch.Tensor = None) -> torch.Tensor:
        """xs: float64 [frames, C] device latents; ts: timesteps; conds: bf16 token tensors."""
        n = len(xs)
        if n > self.max_rows:
            raise ValueError(f"{n} rows > max_rows {self.max_rows}")
        out = self.out if out is None else out
        xp = (ctypes.c_void_p * n)(*[x.data_ptr() for x in xs])
        tp = (ctypes.c_float * n)(*[float(t) for t in ts])
        cp = (ctypes.c_void_p * n)(*[c.data_ptr() for c in conds])
        with self._lock:
            self._order_after_previous_use()
            _native.check(self.lib.rf_dit_forward(self.handle, n, xp, tp, cp, out.data_ptr(),
                                                  _device.current_stream_handle()), "rf_dit_forward")
            self.mark_used()
        return out[:n]


# ------------------------------------------------- StreamPipeline velocity model --
@dataclass(frozen=True)
class _Uncond:
    prompt_hash: int
    hint_strength: float = 0.0
    timbre_strength: float = 0.0


@dataclass
class _Pending:
    xs: list = field(default_factory=list)
    ts: list = field(default_factory=list)
    conds: list = field(default_factory=list)


class DiTVelocity:
    """Velocity-model plug-in for ``StreamPipeline``: the DiT replaces ToyFlowModel.

    Each tick, every active slot contributes one DiT row per condition (+ one
    unconditional row when its guidance step needs a negative); all rows run in ONE
    batched forward, each with its own timestep sigma[step] (north_star (a)).  The
    solver reads the fp32 velocities in place (RF_ROWF_V_F32).
    """

    def __init__(self, dit: DiT, uncond_prompt: int = 0):
        self.dit = dit
        self.uncond_prompt = uncond_prompt
        self._p = _Pending()
        self._last_rows = 0

    @property
    def launches_per_forward(self) -> int:
        """Kernels the last forward launched (counted from its captured CUDA graph)."""
        n = self.dit.lib.rf_dit_launches(self.dit.handle, self._last_rows) if self._last_rows else 0
        return max(n, 0)

    def _row(self, x, t, cond) -> int:
        self._p.xs.append(x)
        self._p.ts.append(t)
        self._p.conds.append(self.dit.cond_tokens(cond.prompt_hash, cond.hint_strength, cond.timbre_strength))
        return len(self._p.xs) - 1

    def _ptr(self, idx) -> int:
        return self.dit.out[idx].data_ptr()

    def prepare_row(self, pipe, slot, row, t_curr: float, need_uncond: bool) -> None:
        conds = slot.request.conditions
        if len(self._p.xs) + len(conds) + int(need_uncond) > self.dit.max_rows:
            raise ValueError("DiT batch exceeds max_rows; raise DiT(max_rows=...)")
        row.n_cond = len(conds)
        for j, c in enumerate(conds):
            row.cond_x0[j] = self._ptr(self._row(slot.x, t_curr, c))
            if len(conds) > 1:
                w = c.weight_device()
                row.cond_w[j] = None if w is None else w.data_ptr()
        if need_uncond:
            row.uncond_x0 = self._ptr(self._row(slot.x, t_curr, _Uncond(self.uncond_prompt)))
        row.flags |= _native.RF_ROWF_COND_V | _native.RF_ROWF_UNCOND_V | _native.RF_ROWF_V_F32

    def forward(self, pipe) -> None:
        p, self._p = self._p, _Pending()
        if p.xs:
            self._last_rows = len(p.xs)
            self.dit.forward(p.xs, p.ts, p.conds)

    def consumed(self, stream) -> None:
        """The pipeline queued the solver that reads this tick's velocities on ``stream``."""
        self.dit.mark_used(stream)

    def reset(self) -> None:
        """Drop rows prepared for a tick that raised before its forward ran."""
        self._p = _Pending()
