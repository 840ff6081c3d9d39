"""Our tcgen05 GEMM vs cuBLAS as K grows (per-tile overhead vs main-loop rate), bf16 out,
weights cycling through 4 copies; 20 back-to-back launches per sample."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import tensor_ops as ops  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


def main():
    for M, N, K in ((3000, 12288, 2048), (3000, 12288, 4096), (3000, 12288, 8192), (8192, 8192, 8192),
                    (3000, 2048, 2048), (12000, 2048, 2048)):
        a = torch.randn(M, K, device="cuda").bfloat16()
        ws = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(2)]
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        bn = 256 if N >= 4096 else 128
        us = timeit(lambda i: ops.gemm(a, ws[i % 2], out=out, epilogue=ops.EPI_BF16, block_n=bn, pair=True))
        cu = timeit(lambda i: torch.matmul(a, ws[i % 2].T, out=out))
        print(f"M={M:5d} N={N:5d} K={K:5d}: ours {us:8.1f} us {fl / us / 1e6:6.0f} TF/s | cuBLAS {cu:8.1f} us "
              f"{fl / cu / 1e6:6.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
