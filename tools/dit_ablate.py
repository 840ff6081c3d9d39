"""In-graph cost of each DiT kernel class: config-2 forwards (4 rows) with one class left out
(RF_DIT_SKIP, read at DiT creation), all variants created in one process (shared weights)
and timed interleaved, round after round, so clocks and thermal state are comparable.
cost = full - ablated.  Timing only (an ablated forward computes garbage).

    python tools/dit_ablate.py [mask ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402

CLASSES = [("full", 0), ("norms x3", 1), ("self-attn", 2), ("cross-attn", 4), ("QKV gemm", 8), ("O gemm", 16),
           ("cross-Q gemm", 32), ("cross-O gemm", 64), ("gate-up gemm", 128), ("down gemm", 256),
           ("norms+self-attn", 3), ("all attention", 6)]


def main():
    masks = [int(x) for x in sys.argv[1:]] or [m for _, m in CLASSES]
    names = {m: n for n, m in CLASSES}
    torch.cuda.set_stream(torch.cuda.Stream())
    cfg = D.DiTConfig()
    base = None
    dits = {}
    for m in masks:
        os.environ["RF_DIT_SKIP"] = str(m)
        dits[m] = D.DiT(cfg, frames=1500, max_rows=4, weights=base.weights if base else None)
        base = base or dits[m]
    os.environ.pop("RF_DIT_SKIP", None)
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(4)]
    ts = [1.0 - 0.1 * i for i in range(4)]
    conds = [base.cond_tokens(i) for i in range(4)]
    for d in dits.values():
        for _ in range(3):
            d.forward(xs, ts, conds)
    torch.cuda.synchronize()
    res = {m: [] for m in masks}
    for _ in range(8):
        for m, d in dits.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(4):
                d.forward(xs, ts, conds)
            b.record()
            torch.cuda.synchronize()
            res[m].append(a.elapsed_time(b) / 4)
    med = {m: sorted(v)[len(v) // 2] for m, v in res.items()}
    full = med.get(0)
    for m in masks:
        extra = f"  saves {full - med[m]:6.3f} ms ({(full - med[m]) / 24 * 1e3:6.1f} us/layer)" if full and m else ""
        print(f"{names.get(m, m)!s:16s} mask {m:4d}: {med[m]:7.3f} ms{extra}", flush=True)


if __name__ == "__main__":
    main()
