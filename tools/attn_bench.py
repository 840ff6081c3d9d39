"""Device time of the tcgen05 attention at the DiT's shapes (self: 750 x 750, cross: 750 x 128;
4 rows, 16 query / 8 KV heads of 128).  RF_ATTN_TWO_PASS=1 selects the earlier kernel."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native  # noqa: E402


def main():
    lib = _native.load()
    lib.rf_attention_tc_bf16.restype = int
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    B, Nq, H, Hk = 4, 750, 16, 8
    for Nk in (750, 128):
        q = torch.randn(B * Nq, H * 128, device="cuda").bfloat16()
        k = torch.randn(B * Nk, Hk * 128, device="cuda").bfloat16()
        pad = (Nk + 7) // 8 * 8
        vt = torch.randn(B, Hk, 128, pad, device="cuda").bfloat16()
        out = torch.empty(B * Nq, H * 128, device="cuda", dtype=torch.bfloat16)

        def run():
            _native.check(lib.rf_attention_tc_bf16(vp(q.data_ptr()), vp(k.data_ptr()), vp(vt.data_ptr()),
                                                   vp(out.data_ptr()), B, Nq, Nk, pad, H, Hk, i64(H * 128),
                                                   i64(Hk * 128), i64(H * 128),
                                                   vp(torch.cuda.current_stream().cuda_stream)), "attn")

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            run()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        fl = 4.0 * B * H * Nq * Nk * 128
        print(f"{'two-pass' if os.environ.get('RF_ATTN_TWO_PASS') else 'single-pass'} Nk={Nk}: {us:7.1f} us "
              f"{fl / us / 1e6:6.0f} TF/s (algorithmic)", flush=True)


if __name__ == "__main__":
    main()
