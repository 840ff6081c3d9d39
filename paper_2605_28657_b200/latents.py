"""Latent primitives: keyed gaussian noise on the GPU, content hashing, latent metrics.

Mirrors reference ``pkg/src/ringflow/latents.py`` (public names at :17-27).  A latent is
a [T, D] frame-major float64 array (latents.py:3-6); on this path it lives on the GPU
as a torch float64 tensor, and the public functions accept numpy arrays or tensors.

``NoiseSource`` derives the same 128-bit Philox key as the reference (blake2b over
(seed, step, stream, tag), latents.py:130-135) on the host and fills the tensor with
the bit-exact numpy ziggurat on the device (``rf_normal_fill``, csrc/rf_noise.cu).
"""
from __future__ import annotations

import ctypes
import hashlib
import struct
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native

__all__ = [
    "Latent",
    "Curve",
    "NoiseSource",
    "NoiseCache",
    "ShapeMismatchError",
    "content_hash",
    "prompt_id",
    "mse",
    "rms_diff",
    "segment_cosine_similarity",
]

Latent = np.ndarray
Curve = np.ndarray

_MASK64 = (1 << 64) - 1


class ShapeMismatchError(ValueError):
    """Operands do not share the shape an operation requires."""


def _shape(a):
    return tuple(a.shape)


def _require_same_shape(a, b) -> None:
    if _shape(a) != _shape(b):
        raise ShapeMismatchError(f"shape mismatch: {_shape(a)} vs {_shape(b)}")


def mse(a, b) -> float:
    """Mean squared element difference (latents.py:42-46), reduced on the GPU.

    The reduction order is fixed (csrc/rf_emit.cu), so identical inputs give exactly
    0.0 and repeated calls are bit-identical; values can differ from numpy's pairwise
    sum in the last ulp.
    """
    _require_same_shape(a, b)
    dev = _device.device()
    ta, tb = _device.to_device_f64(a, dev), _device.to_device_f64(b, dev)
    n = ta.numel()
    if n == 0:
        return float("nan")
    out = torch.empty(1, dtype=torch.float64, device=dev)
    lib = _native.load()
    elems = lib.rf_reduce_workspace_elems(n)
    scratch = _device.workspace(8 * elems, "reduce", dev)   # this stream's own partials
    _native.check(lib.rf_mse(ta.data_ptr(), tb.data_ptr(), n, out.data_ptr(), scratch.data_ptr(), elems,
                             _device.current_stream_handle()), "rf_mse")
    return float(out.item())


def rms_diff(a, b) -> float:
    """sqrt(mse(a, b)) (latents.py:49-51)."""
    return float(np.sqrt(mse(a, b)))


def segment_cosine_similarity(a, b, n_segments: int) -> np.ndarray:
    """Per-segment cosine similarity of flattened frame segments (latents.py:54-77)."""
    _require_same_shape(a, b)
    frames = a.shape[0]
    if n_segments < 1 or n_segments > frames:
        raise ValueError(f"n_segments must be in [1, {frames}], got {n_segments}")
    dev = _device.device()
    ta, tb = _device.to_device_f64(a, dev), _device.to_device_f64(b, dev)
    base = frames // n_segments
    out = np.zeros(n_segments)
    for i in range(n_segments):
        lo = i * base
        hi = (i + 1) * base if i < n_segments - 1 else frames
        u = ta[lo:hi].reshape(-1)
        v = tb[lo:hi].reshape(-1)
        nu = float(torch.linalg.vector_norm(u))
        nv = float(torch.linalg.vector_norm(v))
        if nu == 0.0 or nv == 0.0:
            continue
        out[i] = float(torch.dot(u, v)) / (nu * nv)
    return out


def _feed(h, part) -> None:
    # Same byte encoding as the reference's content hash (latents.py:80-101).
    if isinstance(part, bool):
        part = int(part)
    if isinstance(part, int):
        h.update(b"i" + part.to_bytes(16, "little", signed=True))
    elif isinstance(part, float):
        h.update(b"f" + struct.pack("<d", part))
    elif isinstance(part, str):
        h.update(b"s" + part.encode("utf-8"))
    elif isinstance(part, bytes):
        h.update(b"b" + part)
    elif isinstance(part, torch.Tensor):
        arr = part.detach().to("cpu", torch.float64).contiguous().numpy()
        h.update(b"a" + str(tuple(arr.shape)).encode() + arr.tobytes())
    elif isinstance(part, np.ndarray):
        h.update(b"a" + str(part.shape).encode() + np.ascontiguousarray(part, dtype=np.float64).tobytes())
    elif part is None:
        h.update(b"n")
    elif isinstance(part, (tuple, list)):
        h.update(b"(")
        for p in part:
            _feed(h, p)
        h.update(b")")
    else:
        raise TypeError(f"unhashable content part: {type(part)!r}")


def content_hash(*parts) -> int:
    """Stable 63-bit content hash (latents.py:104-109)."""
    h = hashlib.blake2b(digest_size=8)
    for part in parts:
        _feed(h, part)
    return int.from_bytes(h.digest(), "little") & (2**63 - 1)


def prompt_id(text: str) -> int:
    return content_hash("prompt", text)


_KEY_CACHE: dict = {}


def philox_key(seed: int, stream: int, step: int, tag: str) -> int:
    """128-bit Philox key of a (seed, stream, step, tag) draw (latents.py:130-135)."""
    k = (seed, stream, step, tag)
    key = _KEY_CACHE.get(k)
    if key is None:
        if step < 0:
            raise ValueError("noise step index must be >= 0")
        h = hashlib.blake2b(digest_size=16)
        h.update(struct.pack("<qq", seed, step))
        h.update(stream.to_bytes(16, "little", signed=True))
        h.update(tag.encode("utf-8"))
        key = int.from_bytes(h.digest(), "little")
        if len(_KEY_CACHE) > 1 << 16:
            _KEY_CACHE.clear()
        _KEY_CACHE[k] = key
    return key


def _numel(shape) -> int:
    if isinstance(shape, int):
        return shape
    n = 1
    for s in shape:
        n *= int(s)
    return n


def fill_normals(draws, status: torch.Tensor = None, stream: int = None) -> None:
    """Batched bit-exact normal fill. ``draws`` = [(key, out_tensor_f64), ...] on one device;
    ``stream``: the CUDA stream handle to run on (default: the current stream)."""
    if not draws:
        return
    st = _device.current_stream_handle() if stream is None else stream
    lib = _native.load()
    arr = (_native.RfDraw * len(draws))()
    for i, (key, out) in enumerate(draws):
        arr[i].k0 = key & _MASK64
        arr[i].k1 = key >> 64
        arr[i].n = out.numel()
        arr[i].out = out.data_ptr()
    nbytes = lib.rf_normal_workspace_bytes(arr, len(draws))
    dev = draws[0][1].device
    ws = _device.workspace(nbytes, "noise", dev, st)
    own_status = status is None
    if own_status:
        status = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(lib.rf_normal_fill(arr, len(draws), ws.data_ptr(), ws.numel(), status.data_ptr(), st),
                  "rf_normal_fill")
    if own_status:
        flags = int(status.item())
        if flags & _native.RF_STATUS_NOISE_SHORT:
            raise _native.NativeError("normal fill ran out of stream positions")


class NoiseCache:
    """Device cache of keyed normal draws: philox key -> float64 buffer.

    A draw is a pure function of its key, and the key derives from (seed, content key,
    step, tag) only -- denoise and curves are not in it (reference pipeline.py:95-96,
    latents.py:118-150) -- so a stream regenerating the same request draws the same S x 2 + 1
    tensors every generation.  Entries are LRU within ``capacity_bytes``; an entry used in
    the current tick (``stamp``) is never evicted, so every pointer handed to this tick's
    kernels stays valid (all users run on the owning pipeline's stream, in order).
    """

    def __init__(self, capacity_bytes: int, numel: int, device):
        self.capacity_bytes = int(capacity_bytes)
        self.numel = int(numel)
        self._dev = device
        self._entries: OrderedDict = OrderedDict()   # key -> [tensor, stamp, filled]
        self.hits = 0
        self.misses = 0

    @property
    def bytes(self) -> int:
        return len(self._entries) * self.numel * 8

    def lookup(self, key: int, stamp: int):
        """(buffer, hit): the cached draw for ``key``, or a buffer to fill for it (then
        ``filled`` once its fill is queued; an entry never filled stays a miss)."""
        ent = self._entries.get(key)
        if ent is not None:
            ent[1] = stamp
            self._entries.move_to_end(key)
            if ent[2]:
                self.hits += 1
                return ent[0], True
            self.misses += 1
            return ent[0], False
        self.misses += 1
        buf = None
        nbytes = self.numel * 8
        while self._entries and self.bytes + nbytes > self.capacity_bytes:
            old_key, old = next(iter(self._entries.items()))
            if old[1] >= stamp:          # in use this tick: keep it
                break
            del self._entries[old_key]
            buf = old[0]                 # reuse the evicted buffer (same size)
        if buf is None:
            buf = torch.empty(self.numel, dtype=torch.float64, device=self._dev)
        self._entries[key] = [buf, stamp, False]
        return buf, False

    def filled(self, keys) -> None:
        """Mark entries whose generation has been queued on the owning stream."""
        for key in keys:
            ent = self._entries.get(key)
            if ent is not None:
                ent[2] = True

    def clear(self) -> None:
        self._entries.clear()


@dataclass(frozen=True)
class NoiseSource:
    """Counter-based keyed gaussian noise (latents.py:117-150), generated on the GPU."""

    seed: int
    stream: int = 0

    @staticmethod
    def step_safe(step: int) -> int:
        if step < 0:
            raise ValueError("noise step index must be >= 0")
        return step

    def key(self, step: int, tag: str) -> int:
        return philox_key(self.seed, self.stream, self.step_safe(step), tag)

    def normal_device(self, step: int, tag: str, shape, out: torch.Tensor = None) -> torch.Tensor:
        """Standard-normal float64 tensor on the device for (step, tag)."""
        shp = (shape,) if isinstance(shape, int) else tuple(int(s) for s in shape)
        if out is None:
            out = torch.empty(shp, dtype=torch.float64, device=_device.device())
        fill_normals([(self.key(step, tag), out)])
        return out

    def normal(self, step: int, tag: str, shape) -> np.ndarray:
        """Standard-normal tensor for the given (step, purpose-tag) key (host copy)."""
        return self.normal_device(step, tag, shape).cpu().numpy()

    def uniform_device(self, step: int, tag: str, shape) -> torch.Tensor:
        shp = (shape,) if isinstance(shape, int) else tuple(int(s) for s in shape)
        out = torch.empty(shp, dtype=torch.float64, device=_device.device())
        key = self.key(step, tag)
        lib = _native.load()
        arr = (_native.RfDraw * 1)()
        arr[0].k0, arr[0].k1, arr[0].n, arr[0].out = key & _MASK64, key >> 64, out.numel(), out.data_ptr()
        _native.check(lib.rf_uniform_fill(arr, 1, _device.current_stream_handle()), "rf_uniform_fill")
        return out

    def uniform(self, step: int, tag: str, shape) -> np.ndarray:
        """Uniform [0, 1) tensor for the given (step, purpose-tag) key (host copy)."""
        return self.uniform_device(step, tag, shape).cpu().numpy()
