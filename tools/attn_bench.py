"""Device time of the tcgen05 attention at the DiT's shapes (self: 750 x 750, cross: 750 x 128;
4 rows, 16 query / 8 KV heads of 128).  Kernel variants (rf_attn_set_variant) are timed
interleaved in one process, several rounds, 20 back-to-back launches per sample.

    python tools/attn_bench.py [variant ...]     variant = FA64:POLY, e.g. 1:0 1:4 2:0 0:0"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native  # noqa: E402


def main():
    lib = _native.load()
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    variants = [tuple(int(x) for x in v.split(":")) for v in sys.argv[1:]] or [(1, 6)]
    B, Nq, H, Hk = 4, 750, 16, 8
    for Nk in (750, 128):
        q = torch.randn(B * Nq, H * 128, device="cuda").bfloat16()
        k = torch.randn(B * Nk, Hk * 128, device="cuda").bfloat16()
        pad = (Nk + 7) // 8 * 8
        vt = torch.randn(B, Hk, 128, pad, device="cuda").bfloat16()
        out = torch.empty(B * Nq, H * 128, device="cuda", dtype=torch.bfloat16)
        s = torch.cuda.Stream()
        runs = {}
        for v in variants:
            def run(v=v):
                lib.rf_attn_set_variant(*v)
                _native.check(lib.rf_attention_tc_bf16(vp(q.data_ptr()), vp(k.data_ptr()), vp(vt.data_ptr()),
                                                       vp(out.data_ptr()), B, Nq, Nk, pad, H, Hk, i64(H * 128),
                                                       i64(Hk * 128), i64(H * 128), vp(s.cuda_stream)), "attn")
            for _ in range(3):
                run()
            runs[v] = run
        torch.cuda.synchronize()
        res = {v: [] for v in variants}
        for _ in range(5):
            for v in variants:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                runs[v]()
                a.record(s)
                for _ in range(20):   # back to back: the queue stays ahead of the GPU
                    runs[v]()
                b.record(s)
                torch.cuda.synchronize()
                res[v].append(a.elapsed_time(b) / 20 * 1e3)
        fl = 4.0 * B * H * Nq * Nk * 128
        for v in variants:
            us = sorted(res[v])[len(res[v]) // 2]
            print(f"Nk={Nk} FA64={v[0]} POLY={v[1]}: {us:7.1f} us  {fl / us / 1e6:6.0f} TF/s (algorithmic)", flush=True)


if __name__ == "__main__":
    main()
