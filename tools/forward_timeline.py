"""In-situ timeline of one config-2 DiT forward (4 rows) as it runs in the captured graph at
the power cap: every GEMM launch's CTA entry, work start (after its programmatic-dependency
wait, i.e. when the previous kernel has completed) and exit (globaltimer stamps through
rf_gemm_set_trace_seq).  The non-GEMM kernels between two GEMMs (attention, norms) show as the
gap from one GEMM's last exit to the next GEMM's work start.  Prints per-kind mean durations
over the 24 layers and the forward's total.  python tools/forward_timeline.py"""
import ctypes
import os
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402


def main():
    torch.cuda.set_stream(torch.cuda.Stream())
    cfg = D.DiTConfig()
    dit = D.DiT(cfg, frames=1500, max_rows=4)
    lib = dit.lib
    lib.rf_gemm_set_trace_seq.restype = ctypes.c_int64
    blk = 400 * 16 * 8
    maxl = 400
    buf = torch.zeros(maxl * blk, dtype=torch.int64, device="cuda")
    lib.rf_gemm_set_trace_seq(ctypes.c_void_p(buf.data_ptr()), ctypes.c_int64(maxl))
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(4)]
    ts = [1.0 - 0.1 * i for i in range(4)]
    conds = [dit.cond_tokens(i) for i in range(4)]
    dit.forward(xs, ts, conds)            # direct launches, then the graph capture
    torch.cuda.synchronize()
    lib.rf_gemm_set_trace_seq(ctypes.c_void_p(0), ctypes.c_int64(0))
    t0 = time.time()
    while time.time() - t0 < 1.5:         # into the power-capped steady state
        dit.forward(xs, ts, conds)
    buf.zero_()
    dit.forward(xs, ts, conds)
    torch.cuda.synchronize()
    t = buf.view(maxl, 400, 16, 8).cpu().numpy()
    launches = [i for i in range(maxl) if t[i, :, 15, 7].max() > 0]
    rows = []
    for i in launches:
        ent = t[i, :, 15, 7]
        work = t[i, :, 13, 7]
        ex = t[i, :, 14, 7]
        live = ent > 0
        rows.append((ent[live].min(), work[live].min(), ex[live].max()))
    base = rows[0][0]
    n = len(rows)
    per = (n - 7) // 24                   # 6 prologue GEMMs, 6 per layer, 1 output GEMM
    names = ["qkv", "o", "xq+xattn", "o_cross", "gate_up", "down"]
    dur, gap = defaultdict(list), defaultdict(list)
    for li in range(24):
        for k in range(per):
            idx = 6 + li * per + k
            s, w, e = rows[idx]
            dur[names[k]].append((e - w) / 1e3)
            pe = rows[idx - 1][2]
            gap["before " + names[k]].append((w - pe) / 1e3)
    print(f"{n} GEMM launches traced; forward {(rows[-1][2] - base) / 1e3:.1f} us "
          f"(first GEMM entry to last GEMM exit)")
    for k in names:
        print(f"  {k:10s} work {sum(dur[k]) / len(dur[k]):7.2f} us   gap before {sum(gap['before ' + k]) / 24:6.2f} us")
    print("  (gap before qkv = norm1 (+ launch); before o = self-attention; before gate_up = norm3; "
          "before o_cross = 0 (xattn fused); before xq+xattn: the O-proj -> cross-Q handoff)")
    # per-tile clock64 stamps of the same launches (MMA warp of the leader CTAs: 0 tile start,
    # 1 accumulator free, 2 first operands, 3 all k blocks issued; epilogue warp: 4 accumulator
    # full, 5 done) -- is each GEMM kind fed, or waiting for its epilogue?
    print("  per tile (cycles, mean over layers):  acc-wait  operand-wait  issue-span  epilogue")
    for k in range(per):
        aw, ow, sp, ep = [], [], [], []
        for li in range(24):
            blk_ = t[launches[6 + li * per + k]]
            for c in range(400):
                for it in range(16):
                    st = blk_[c, it]
                    if st[0] and st[1] and st[2] and st[3]:
                        aw.append(st[1] - st[0])
                        ow.append(st[2] - st[1])
                        sp.append(st[3] - st[2])
                    if st[4] and st[5]:
                        ep.append(st[5] - st[4])
        m = lambda v: sum(v) / len(v) if v else float("nan")  # noqa: E731
        print(f"  {names[k]:10s} {m(aw):9.0f} {m(ow):13.0f} {m(sp):11.0f} {m(ep):9.0f}")
    # QKV: epilogue by column block kind (tile = unit + k * 74, 12 m-blocks, 16 n-blocks of
    # 256: Q 0-7 with RoPE, K 8-11 with RoPE, V 12-15 written transposed)
    kinds = {"q": [], "k": [], "v": []}
    for li in range(24):
        blk_ = t[launches[6 + li * per]]
        for c in range(0, 400):
            for it in range(16):
                st = blk_[c, it]
                if st[4] and st[5]:
                    tile = (c >> 1) + it * 74
                    nb = tile // 12
                    kinds["q" if nb < 8 else "k" if nb < 12 else "v"].append(st[5] - st[4])
    print("  qkv epilogue by block kind: " + ", ".join(f"{k} {sum(v) / max(len(v), 1):.0f} cycles (n={len(v)})"
                                                      for k, v in kinds.items()))


if __name__ == "__main__":
    main()
