"""Device time of the tcgen05 GEMM on the DiT's shapes, one CTA per tile vs CTA pairs.

    python tools/gemm_bench.py
Median of 20 back-to-back launches (weights cycle through 4 copies > L2 so B is read
from HBM as in the forward, where every layer has its own weights)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import tensor_ops as ops  # noqa: E402

SHAPES = [("qkv", 4096, 2048), ("o/qc/oc", 2048, 2048), ("gate-up", 12288, 2048), ("down", 2048, 6144),
          ("kv-cross", 2048, 2048, 512)]


def main():
    M0 = 3000
    for sh in SHAPES:
        name, N, K = sh[:3]
        M = sh[3] if len(sh) > 3 else M0
        a = torch.randn(M, K, device="cuda").bfloat16()
        ws = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(4)]
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        res = []
        for bn in (128, 256):
            for pair in (False, True):
                for _ in range(3):
                    ops.gemm(a, ws[0], out=out, epilogue=ops.EPI_BF16, block_n=bn, pair=pair)
                torch.cuda.synchronize()
                ts = []
                for i in range(20):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    ops.gemm(a, ws[i % 4], out=out, epilogue=ops.EPI_BF16, block_n=bn, pair=pair)
                    e.record()
                    torch.cuda.synchronize()
                    ts.append(s.elapsed_time(e) * 1e3)
                us = sorted(ts)[len(ts) // 2]
                res.append(f"bn={bn} pair={int(pair)}: {us:7.1f} us {fl / us / 1e6:6.0f} TF/s")
        # cuBLAS (torch.matmul, bf16 out) on the same shape, for reference only
        o16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for _ in range(3):
            torch.matmul(a, ws[0].T, out=o16)
        torch.cuda.synchronize()
        ts = []
        for i in range(20):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch.matmul(a, ws[i % 4].T, out=o16)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        us = sorted(ts)[len(ts) // 2]
        res.append(f"cuBLAS: {us:7.1f} us {fl / us / 1e6:6.0f} TF/s")
        print(f"{name:9s} M={M} N={N} K={K} | " + " | ".join(res), flush=True)


if __name__ == "__main__" and "--epi" not in sys.argv:
    main()


def epilogues():
    """Same pair-tile GEMM, different epilogues (O-proj and down-proj shapes)."""
    for N, K in ((2048, 2048), (2048, 6144)):
        M = 3000
        a = torch.randn(M, K, device="cuda").bfloat16()
        ws = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(4)]
        h = torch.randn(M, N, device="cuda")
        gate = torch.randn(4, N, device="cuda")
        o16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        o32 = torch.empty(M, N, device="cuda")
        fl = 2.0 * M * N * K
        res = []
        for name, kw in (("bf16", dict(out=o16, epilogue=ops.EPI_BF16)), ("f32", dict(out=o32, epilogue=ops.EPI_F32)),
                         ("resid", dict(out=h, epilogue=ops.EPI_RESID_GATE, gate=gate, rows_per_batch=750))):
            for _ in range(3):
                ops.gemm(a, ws[0], block_n=128, pair=True, **kw)
            torch.cuda.synchronize()
            ts = []
            for i in range(20):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                ops.gemm(a, ws[i % 4], block_n=128, pair=True, **kw)
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
            us = sorted(ts)[len(ts) // 2]
            res.append(f"{name}: {us:6.1f} us {fl / us / 1e6:5.0f} TF/s")
        print(f"epilogues M={M} N={N} K={K} pair bn=128 | " + " | ".join(res), flush=True)


if __name__ == "__main__" and "--epi" in sys.argv:
    epilogues()
