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
