"""256 x 256 pair tiles vs 512 x 256 pair tiles (two m-subtiles per CTA) on the DiT's GEMM
shapes at M = 3000 (4 rows x 750 tokens), against cuBLAS (torch.matmul, bf16 out).

    python tools/gemm_mt_bench.py
Mean of 40 back-to-back launches (weights cycle through 4 copies > L2, as in the forward,
where every layer has its own weights)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import tensor_ops as ops  # noqa: E402

SHAPES = [("gate-up swiglu", 12288, 2048, ops.EPI_SWIGLU), ("gate-up bf16", 12288, 2048, ops.EPI_BF16),
          ("qkv bf16", 4096, 2048, ops.EPI_BF16), ("o bf16", 2048, 2048, ops.EPI_BF16),
          ("down bf16", 2048, 6144, ops.EPI_BF16)]


def timed(fn, n=40):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(n):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / n


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    for name, N, K, epi in SHAPES:
        a = torch.randn(M, K, device="cuda").bfloat16()
        ws = [(torch.randn(N, K, device="cuda") * 0.02).bfloat16() for _ in range(4)]
        out = torch.empty(M, N // 2 if epi == ops.EPI_SWIGLU else N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        line = [f"{name:15s} M={M} N={N:5d} K={K}:"]
        for bn, mt in ((128, 1), (256, 1), (256, 2)):
            us = timed(lambda i: ops.gemm(a, ws[i % 4], out=out, epilogue=epi, block_n=bn, pair=True,
                                          m_subtiles=mt))
            line.append(f"{bn}x{mt}: {us:6.1f} us {fl / us / 1e6:5.0f} TF/s")
        o16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        us = timed(lambda i: torch.matmul(a, ws[i % 4].T, out=o16))
        line.append(f"cuBLAS: {us:6.1f} us {fl / us / 1e6:5.0f} TF/s")
        print(" | ".join(line), flush=True)


if __name__ == "__main__":
    main()
