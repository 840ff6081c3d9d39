"""Thin Python handles on the tensor-core kernels (tcgen05 GEMM, attention, norms).

These are the building blocks of the DiT velocity model (``dit.py``); each call is one
launch of a hand-written sm_100a kernel through the C ABI.  Tensors are torch CUDA
tensors (memory and streams only).
"""
from __future__ import annotations

import torch

from . import _device, _native

EPI_BF16, EPI_F32, EPI_RESID_GATE, EPI_SWIGLU, EPI_F32_SCALE = 0, 1, 2, 3, 4


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor = None, epilogue: int = EPI_BF16,
         gate: torch.Tensor = None, rows_per_batch: int = 1, alpha: float = 1.0, block_n: int = None,
         pair: bool = False):
    """out = a @ b.T with a [M, K] bf16 and b [N, K] bf16 (K-major), fp32 accumulation.

    ``pair``: 256 x block_n tiles on a CTA pair (tcgen05 cta_group::2) instead of 128 x block_n
    tiles on one CTA."""
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16 and a.is_cuda and b.is_cuda
    M, K = a.shape
    N = b.shape[0]
    assert b.shape[1] == K and a.stride(1) == 1 and b.stride(1) == 1
    if block_n is None:
        block_n = 256 if N % 256 == 0 else 128
    if out is None:
        if epilogue == EPI_BF16:
            out = torch.empty(M, N, dtype=torch.bfloat16, device=a.device)
        elif epilogue == EPI_SWIGLU:
            out = torch.empty(M, N // 2, dtype=torch.bfloat16, device=a.device)
        else:
            out = torch.zeros(M, N, dtype=torch.float32, device=a.device)
    lib = _native.load()
    _native.check(lib.rf_gemm_bf16(
        a.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K, a.stride(0), b.stride(0), out.stride(0),
        epilogue, gate.data_ptr() if gate is not None else None,
        gate.stride(0) if gate is not None else 0, rows_per_batch, alpha,
        -block_n if pair else block_n,
        _device.current_stream_handle()), "rf_gemm_bf16")
    return out
