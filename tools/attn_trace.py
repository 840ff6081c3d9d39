"""Timeline of the single-pass attention (clock64 stamps from rf_attn_set_trace):
per tile, the softmax time of each head and the MMA gaps.  Self-attention shape."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native  # noqa: E402


def main():
    lib = _native.load()
    lib.rf_attention_tc_bf16.restype = int
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    B, Nq, H, Hk, Nk = 4, 750, 16, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 750
    q = torch.randn(B * Nq, H * 128, device="cuda").bfloat16()
    k = torch.randn(B * Nk, Hk * 128, device="cuda").bfloat16()
    pad = (Nk + 7) // 8 * 8
    vt = torch.randn(B, Hk, 128, pad, device="cuda").bfloat16()
    out = torch.empty(B * Nq, H * 128, device="cuda", dtype=torch.bfloat16)
    nq, ncta = (Nq + 127) // 128, (Nq + 127) // 128 * B * H // (1 if os.environ.get("RF_ATTN_FA64", "1") == "1" else 2)
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
    nt = (Nk + 127) // 128
    for c in (0, 1, ncta // 2):
        t0 = t[c, 4, 0]
        print(f"cta {c}: (cycles from head-0 S(0) ready)")
        for j in range(nt):
            row = []
            for a in range(2):
                s_rdy, p_done, pv, s_iss = t[c, 4 + a, j], t[c, 6 + a, j], t[c, a, j], t[c, 2 + a, j]
                row.append(f"h{a}: S_iss {s_iss - t0 if s_iss else float('nan'):7.0f} S_rdy {s_rdy - t0:7.0f} "
                           f"P_done {p_done - t0:7.0f} (softmax {p_done - s_rdy:5.0f}) PV_iss {pv - t0:7.0f}")
            print(f"  j={j}  " + " | ".join(row))
    soft = (t[:, 6:8, :nt] - t[:, 4:6, :nt]).ravel()
    lat = (t[:, 4:6, 1:nt] - t[:, 2:4, 1:nt]).ravel()
    gap = (t[:, 2:4, 1:nt] - t[:, 0:2, 0:nt - 1]).ravel()
    g0, g1 = t[:, 0, 15], t[:, 1, 15]
    print(f"kernel span {(g1.max() - g0.min()) / 1e3:.1f} us; CTA durations median {np.median(g1 - g0) / 1e3:.1f} us "
          f"max {np.max(g1 - g0) / 1e3:.1f}; start offsets: {np.percentile(g0 - g0.min(), [0, 50, 75, 90, 100]) / 1e3}")
    for name, a, b in (("wait->S loaded", 4, 8), ("S loaded->max done", 8, 10), ("exps+stores issued", 10, 12),
                       ("st_wait+arrive", 12, 6)):
        d = np.concatenate([(t[:, b + h, :nt - 1] - t[:, a + h, :nt - 1]).ravel() for h in range(2)])
        print(f"  {name:22s} median {np.median(d):6.0f} cyc")
    print(f"median softmax per head-tile {np.median(soft):.0f} cyc; S issue->ready {np.median(lat):.0f}; "
          f"PV issue->S issue {np.median(gap):.0f}; CTA span {np.median(t[:, 6:8, nt - 1].max(1) - t[:, 4, 0]):.0f}")


if __name__ == "__main__":
    main()
