"""Per-CTA timeline of the self-attention kernel (rf_attn_fa64_kernel<1>) at config-2 shape
from its in-kernel stamps (rf_attn_set_trace; debugging hook, null in production):
CTA entry / exit (globaltimer), SM id, and per key tile (clock64) S-ready, S loaded,
exponentials done and P published for the softmax, PV / S issue for the MMA warp.
python tools/attn_trace.py [B N]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
N = int(sys.argv[2]) if len(sys.argv) > 2 else 750
H, Hk = 16, 8
lib = _native.load()
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(B * N, H * 128, device="cuda", generator=g).bfloat16()
k = torch.randn(B * N, Hk * 128, device="cuda", generator=g).bfloat16()
npad = (N + 7) // 8 * 8
vt = torch.randn(B, Hk, 128, npad, device="cuda", generator=g).bfloat16()
out = torch.empty(B * N, H * 128, device="cuda", dtype=torch.bfloat16)
vp, i64 = ctypes.c_void_p, ctypes.c_int64
st = torch.cuda.current_stream().cuda_stream
nq = (N + 127) // 128
ncta = nq * B * H
nt = (N + 63) // 64


def run():
    _native.check(lib.rf_attention_tc_bf16(vp(q.data_ptr()), vp(k.data_ptr()), vp(vt.data_ptr()), vp(out.data_ptr()),
                                           B, N, N, npad, H, Hk, i64(H * 128), i64(Hk * 128), i64(H * 128), vp(st)),
                  "attn")


for _ in range(5):
    run()
buf = torch.zeros(ncta * 16 * 16, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
rows = []
for rep in range(3):
    buf.zero_()
    flush.fill_(1)
    _native.check(lib.rf_attn_set_trace(vp(buf.data_ptr())), "trace")
    run()
    torch.cuda.synchronize()
    _native.check(lib.rf_attn_set_trace(vp(0)), "trace")
    rows.append(buf.cpu().numpy().reshape(ncta, 16, 16).astype(np.int64))
tr = rows[-1]
t0, t1 = tr[:, 0, 15], tr[:, 1, 15]
sm, c0, c1 = tr[:, 3, 15], tr[:, 3, 14], tr[:, 3, 13]
base = t0.min()
dur = (t1 - t0) / 1e3
print(f"B={B} N={N}: {ncta} CTAs, {nt} key tiles each; kernel span {(t1.max() - base) / 1e3:.2f} us")
order = np.argsort(t0)
start_us = (t0 - base) / 1e3
wave1 = start_us < 1.0
print(f"CTAs starting in the first us: {wave1.sum()}  later: {(~wave1).sum()}")
for name, m in (("first wave", wave1), ("later", ~wave1)):
    if m.any():
        print(f"  {name:10s} start {start_us[m].min():6.2f}-{start_us[m].max():6.2f} us  duration mean {dur[m].mean():6.2f} "
              f"min {dur[m].min():6.2f} max {dur[m].max():6.2f} us  end max {((t1[m] - base) / 1e3).max():6.2f}")
# per-SM occupancy: CTAs per SM and their spans
per_sm = {}
for i in range(ncta):
    per_sm.setdefault(int(sm[i]), []).append(i)
cnt = np.bincount([len(v) for v in per_sm.values()])
print("CTAs per SM histogram:", {i: int(c) for i, c in enumerate(cnt) if c})
# clock-domain per-tile breakdown for head 0 (events: 4 S ready, 8 S loaded, 12 exps done, 6 P published,
# 0 PV issued, 2 S issued)
clk = lambda ev: tr[:, ev, :min(nt, 15)].astype(np.float64)
ghz = ((c1 - c0) / np.maximum(t1 - t0, 1)).mean()
print(f"SM clock from stamps: {ghz:.3f} GHz")
s_ready, s_load, exp_done, p_pub = clk(4), clk(8), clk(12), clk(6)
first = (s_ready[:, 0] - c0) / ghz / 1e3
print(f"entry -> S(0) ready: mean {first.mean():.2f} us  (Q + first K load, S MMA)")
last = min(nt, 15) - 1
tail = (c1 - p_pub[:, last]) / ghz / 1e3
print(f"P(last) -> exit: mean {tail.mean():.2f} us  (last PV, O read, normalise, store)")
sm_cyc = (exp_done - s_ready)[:, 1:last]
ld = (s_load - s_ready)[:, 1:last]
pub = (p_pub - exp_done)[:, 1:last]
gap = (s_ready[:, 2:last + 1] - p_pub[:, 1:last])
print(f"per tile (cycles, tiles 1..{last - 1}): S ready -> loaded {ld.mean():.0f}, S ready -> exps done {sm_cyc.mean():.0f}, "
      f"exps done -> P published (st wait + barrier) {pub.mean():.0f}, P published -> next S ready {gap.mean():.0f}")
for name, m in (("first wave", wave1), ("later", ~wave1)):
    if m.any():
        per_tile = ((p_pub[m, last] - p_pub[m, 1]) / (last - 1)).mean()
        print(f"  {name}: {per_tile:.0f} cycles per key tile in steady state")
