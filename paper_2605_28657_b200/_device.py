"""Device plumbing: the CUDA device, streams, workspaces and host<->device conversion.

PyTorch is used only for device memory and streams; all arithmetic on the hot path is
done by the sm_100a kernels in ``csrc/`` through the C ABI.  There is no CPU fallback:
without a CUDA device every compute entry point raises.
"""
from __future__ import annotations

import threading

import numpy as np
import torch

from . import _native

_ws_lock = threading.Lock()
_workspaces: dict = {}


class NoDeviceError(RuntimeError):
    pass


_checked = False


def device() -> torch.device:
    global _checked
    if not _checked:   # availability and the library are checked once per process
        if not torch.cuda.is_available():
            raise NoDeviceError(
                "paper_2605_28657_b200 computes only on a CUDA device (sm_100a); none is available"
            )
        _native.load()
        _checked = True
    return torch.device("cuda", torch.cuda.current_device())


class on_stream:
    """``with on_stream(s):`` makes ``s`` torch's current stream -- the same effect as
    ``torch.cuda.stream(s)`` for a stream on the current device, at a fraction of its host
    cost (the pipeline enters it on every tick)."""

    __slots__ = ("_stream", "_args", "_prev", "_ctx")

    def __init__(self, stream: torch.cuda.Stream):
        self._stream = stream
        self._args = (stream.stream_id, stream.device_index, stream.device_type)
        self._ctx = None

    def __enter__(self):
        if torch._C._cuda_getDevice() != self._args[1]:
            self._ctx = torch.cuda.stream(self._stream)   # other device: the full switch
            return self._ctx.__enter__()
        self._prev = torch._C._cuda_getCurrentStream(self._args[1])
        torch._C._cuda_setStream(stream_id=self._args[0], device_index=self._args[1], device_type=self._args[2])
        return self._stream

    def __exit__(self, *exc):
        if self._ctx is not None:
            return self._ctx.__exit__(*exc)
        p = self._prev
        torch._C._cuda_setStream(stream_id=p[0], device_index=p[1], device_type=p[2])
        return False


def current_stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_device_f64(x, dev=None) -> torch.Tensor:
    """Contiguous float64 device tensor view/copy of a numpy array or tensor."""
    dev = dev or device()
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=torch.float64)
    else:
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        if not a.flags.writeable:   # read-only views (CompletionRecord.latent): torch needs a writable buffer
            a = a.copy()
        t = torch.from_numpy(a).to(dev)
    return t.contiguous()


def to_host(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def workspace(nbytes: int, tag: str = "default", dev=None, stream: int = None) -> torch.Tensor:
    """A cached uint8 device buffer of at least ``nbytes`` for the work of one stream (the
    current stream unless a stream handle is given)."""
    dev = dev or device()
    key = (dev.index, tag, torch.cuda.current_stream(dev).cuda_stream if stream is None else stream)
    with _ws_lock:
        buf = _workspaces.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
            _workspaces[key] = buf
        return buf
