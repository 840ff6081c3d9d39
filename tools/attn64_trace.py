"""Timeline of the 64-key self-attention kernel with one head per CTA (RF_ATTN_FA64=1):
per key tile, when K/V loads were issued, when S was issued / ready, the softmax phases
and the PV issue, from clock64 stamps (rf_attn_set_trace)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native  # noqa: E402


def main():
    os.environ["RF_ATTN_FA64"] = "1"
    lib = _native.load()
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    B, Nq, H, Hk, Nk = 4, 750, 16, 8, 750
    q = torch.randn(B * Nq, H * 128, device="cuda").bfloat16()
    k = torch.randn(B * Nk, Hk * 128, device="cuda").bfloat16()
    pad = (Nk + 7) // 8 * 8
    vt = torch.randn(B, Hk, 128, pad, device="cuda").bfloat16()
    out = torch.empty(B * Nq, H * 128, device="cuda", dtype=torch.bfloat16)
    ncta = (Nq + 127) // 128 * B * H
    buf = torch.zeros(ncta * 16 * 16, dtype=torch.int64, device="cuda")

    def run():
        _native.check(lib.rf_attention_tc_bf16(vp(q.data_ptr()), vp(k.data_ptr()), vp(vt.data_ptr()),
                                               vp(out.data_ptr()), B, Nq, Nk, pad, H, Hk, i64(H * 128),
                                               i64(Hk * 128), i64(H * 128),
                                               vp(torch.cuda.current_stream().cuda_stream)), "attn")

    for _ in range(3):
        run()
    lib.rf_attn_set_trace(vp(buf.data_ptr()))
    run()
    torch.cuda.synchronize()
    lib.rf_attn_set_trace(vp(0))
    t = buf.cpu().numpy().reshape(ncta, 16, 16).astype(np.float64)
    nt = (Nk + 63) // 64
    names = {13: "K_ld", 14: "V_ld", 2: "S_iss", 4: "S_rdy", 8: "S_in_reg", 10: "O_ok", 12: "exps", 6: "P_done",
             0: "PV_iss"}
    for c in (0, 1, ncta // 2):
        t0 = t[c, 4, 0]
        print(f"cta {c}: cycles from S(0) ready")
        for j in range(nt):
            print("  j=%2d " % j + " ".join(f"{n}={t[c, e, j] - t0:7.0f}" if t[c, e, j] else f"{n}=      -"
                                           for e, n in names.items()))
    d = lambda e1, e0, lo=1: np.median((t[:, e1, lo:nt - 1] - t[:, e0, lo:nt - 1]).ravel())
    print(f"median per tile: S_rdy->S_in_reg {d(8, 4):.0f}  S_in_reg->O_ok {d(10, 8):.0f}  O_ok->exps {d(12, 10):.0f}  "
          f"exps->P_done {d(6, 12):.0f}  P_done->PV_iss {d(0, 6):.0f}")
    per_tile = np.median((t[:, 4, 2:nt - 1] - t[:, 4, 1:nt - 2]).ravel())
    wait_s = np.median((t[:, 4, 1:nt - 1] - t[:, 6, 0:nt - 2]).ravel())
    print(f"tile period {per_tile:.0f} cyc; softmax waiting for S after previous P {wait_s:.0f} cyc")
    g0, g1 = t[:, 0, 15], t[:, 1, 15]
    print(f"kernel span {(g1.max() - g0.min()) / 1e3:.1f} us; CTA durations median {np.median(g1 - g0) / 1e3:.1f} us; "
          f"start offsets pct [0,50,75,90,100] {np.percentile(g0 - g0.min(), [0, 50, 75, 90, 100]) / 1e3}")


if __name__ == "__main__":
    main()
