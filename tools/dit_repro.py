"""Reproducibility probe: a DiT forward sequence with varying row counts (as in the ring's
warm-up), run twice with identical inputs; prints per-call max |diff| between the runs, per
attention variant (rf_attn_set_variant before the DiT -- and its graphs -- are created)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native, dit as D  # noqa: E402


def main():
    torch.cuda.set_stream(torch.cuda.Stream())
    lib = _native.load()
    cfg = D.DiTConfig()
    seq = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "1,2,3,4,4,4,2,4".split(","))]
    base = None
    for v in [tuple(int(y) for y in x.split(":")) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0:0", "1:0", "3:0"])]:
        lib.rf_attn_set_variant(*v)
        dit = D.DiT(cfg, frames=1500, max_rows=4, weights=base.weights if base else None)
        base = base or dit
        conds = [dit.cond_tokens(100 + i) for i in range(4)]
        runs = []
        for rep in range(2):
            outs = []
            for k, n in enumerate(seq):
                g = torch.Generator(device="cuda").manual_seed(1000 + k)
                xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(n)]
                ts = [1.0 - 0.11 * i - 0.01 * k for i in range(n)]
                outs.append(dit.forward(xs, ts, conds[:n]).clone())
            torch.cuda.synchronize()
            runs.append(outs)
        diffs = [(a - b).abs().max().item() for a, b in zip(*runs)]
        fin = all(torch.isfinite(o).all().item() for o in runs[0] + runs[1])
        print(f"variant {v}: finite={fin} per-call max|run1-run2| = {['%.2e' % d for d in diffs]}", flush=True)
        del dit
    lib.rf_attn_set_variant(-1, -1)


if __name__ == "__main__":
    main()
