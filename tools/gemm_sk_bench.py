"""Static persistent tile walk vs stream-K (equal k-block shares per CTA pair) on the DiT's
GEMM shapes at M = 3000 (4 rows x 750 tokens), against cuBLAS (torch.matmul, bf16 out).

    python tools/gemm_sk_bench.py [M]
Mean of 40 back-to-back launches (weights cycle through 4 copies > L2, as in the forward,
where every layer has its own weights)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import tensor_ops as ops  # noqa: E402

SHAPES = [("gate-up swiglu", 12288, 2048, ops.EPI_SWIGLU, 256), ("qkv bf16", 4096, 2048, ops.EPI_BF16, 256),
          ("o bf16", 2048, 2048, ops.EPI_BF16, 128), ("o resid", 2048, 2048, ops.EPI_RESID_GATE, 128),
          ("down bf16", 2048, 6144, ops.EPI_BF16, 128), ("down resid", 2048, 6144, ops.EPI_RESID_GATE, 128)]
# columns: st = static persistent walk, SK = stream-K; 128 / 256 = tile width; then TF/s


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
    for name, N, K, epi, bn in SHAPES:
        a = torch.randn(M, K, device="cuda").bfloat16()
        ws = [(torch.randn(N, K, device="cuda") * 0.02).bfloat16() for _ in range(4)]
        if epi == ops.EPI_RESID_GATE:
            out = torch.zeros(M, N, device="cuda")
            kw = dict(gate=torch.randn(4, N, device="cuda"), rows_per_batch=(M + 3) // 4)
        else:
            out = torch.empty(M, N // 2 if epi == ops.EPI_SWIGLU else N, device="cuda", dtype=torch.bfloat16)
            kw = {}
        fl = 2.0 * M * N * K
        line = [f"{name:15s} M={M} N={N:5d} K={K}:"]
        for bn in (128, 256):
            for sk in (False, True):
                us = timed(lambda i: ops.gemm(a, ws[i % 4], out=out, epilogue=epi, block_n=bn, pair=True,
                                              stream_k=sk, **kw))
                line.append(f"{'SK' if sk else 'st'}{bn}: {us:6.1f} us {fl / us / 1e6:5.0f}")
        o16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        us = timed(lambda i: torch.matmul(a, ws[i % 4].T, out=o16))
        line.append(f"cuBLAS: {us:6.1f} us {fl / us / 1e6:5.0f} TF/s")
        print(" | ".join(line), flush=True)


if __name__ == "__main__":
    main()
