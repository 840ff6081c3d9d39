"""Drive individual hot kernels for ncu / timing (no pipeline bookkeeping around them).

    python tools/prof_kernels.py [decode|noise|all] [--iters N]
Prints CUDA-event timings (warm, L2 flushed between iterations) per case.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_28657_b200 as rf  # noqa: E402
from paper_2605_28657_b200.latents import fill_normals, philox_key  # noqa: E402


def timed(fn, iters, flush, reps=10):
    """Median device time (us) of one fn() call: `reps` calls captured in a CUDA graph
    (no host launch gaps), L2 flushed before each replay."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="?", default="all")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if a.what in ("decode", "all"):
        codec = rf.ToyCodec(channels=64, hop=1920)
        lat = torch.randn(1500, 64, dtype=torch.float64, device=dev) * 0.5
        print("decode 3s window + ov15 (us):", timed(lambda: codec.decode_device(lat, 1425, 1500, 15, False), a.iters, flush))
        print("decode 15s window + ov15 (us):", timed(lambda: codec.decode_device(lat, 1125, 1500, 15, False), a.iters, flush))
        print("decode full 60s (us):", timed(lambda: codec.decode_device(lat, 0, 1500, 0, True), a.iters, flush))
        lat240 = torch.randn(6000, 64, dtype=torch.float64, device=dev) * 0.5
        print("decode full 240s (us):", timed(lambda: codec.decode_device(lat240, 0, 6000, 0, True), a.iters, flush))
    if a.what in ("gemm", "all"):
        from paper_2605_28657_b200 import tensor_ops as ops
        for (M, N, K) in ((3000, 4096, 2048), (3000, 2048, 2048), (3000, 12288, 2048), (3000, 2048, 6144),
                          (6000, 12288, 2048), (8192, 8192, 8192)):
            A = torch.randn(M, K, device=dev).bfloat16()
            B = torch.randn(N, K, device=dev).bfloat16()
            for bn in (128, 256):
                o = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
                us = timed(lambda: ops.gemm(A, B, out=o, block_n=bn), a.iters, flush)
                print(f"gemm {M}x{N}x{K} BN={bn}: {us:8.1f} us  {2*M*N*K/us/1e6:7.1f} TFLOP/s")
            us = timed(lambda: torch.matmul(A, B.T), a.iters, flush)
            print(f"cublas {M}x{N}x{K}:      {us:8.1f} us  {2*M*N*K/us/1e6:7.1f} TFLOP/s")
    if a.what in ("noise", "all"):
        for nd, n in ((1, 96000), (8, 96000), (16, 96000)):
            outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(nd)]
            draws = [(philox_key(1, i, 3, "sde"), o) for i, o in enumerate(outs)]
            st = torch.zeros(1, dtype=torch.int32, device=dev)
            print(f"noise {nd} x {n} (us):", timed(lambda: fill_normals(draws, st), a.iters, flush))


if __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] == "epi"):
    main()


def epilogues():
    from paper_2605_28657_b200 import tensor_ops as ops
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    M, N, K = 3000, 2048, 2048
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(N, K, device=dev).bfloat16()
    x = torch.zeros(M, N, device=dev)
    gate = torch.randn(4, N, device=dev)
    for name, kw in (("f32", dict(epilogue=ops.EPI_F32, out=x)),
                     ("resid_gate", dict(epilogue=ops.EPI_RESID_GATE, out=x, gate=gate, rows_per_batch=750)),
                     ("bf16", dict(epilogue=ops.EPI_BF16))):
        us = timed(lambda: ops.gemm(A, B, block_n=256, **kw), 10, flush)
        print(f"epilogue {name}: {us:.1f} us")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "epi":
    epilogues()
