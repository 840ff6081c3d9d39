"""A/B timing of two DiT configurations that differ only in an environment switch read at
rf_dit_create (e.g. RF_DIT_L2_PERSIST=0): both share one set of weights, forwards alternate
in rounds so clock / power drift hits both equally.  Median ms per forward (CUDA graph).

    python tools/dit_ab.py VAR=VALUE [rows]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402


def main():
    var, val = sys.argv[1].split("=", 1)
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    torch.cuda.set_stream(torch.cuda.Stream())
    cfg = D.DiTConfig()
    base = D.DiT(cfg, frames=1500, max_rows=rows)
    os.environ[var] = val
    alt = D.DiT(cfg, frames=1500, max_rows=rows, weights=base.weights)
    del os.environ[var]
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(rows)]
    ts = [1.0 - 0.1 * i for i in range(rows)]
    conds = [base.cond_tokens(i) for i in range(rows)]
    ya = base.forward(xs, ts, conds).clone()
    yb = alt.forward(xs, ts, conds).clone()
    print(f"outputs identical: {torch.equal(ya, yb)}  max|diff| {(ya - yb).abs().max().item():.3e}")
    res = {"default": [], f"{var}={val}": []}
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(8):
        for name, m in (("default", base), (f"{var}={val}", alt)):
            for _ in range(3):
                m.forward(xs, ts, conds)
            a.record()
            for _ in range(10):
                m.forward(xs, ts, conds)
            b.record()
            torch.cuda.synchronize()
            res[name].append(a.elapsed_time(b) / 10)
    fl = cfg.flops_per_forward(rows, 1500)
    for k, v in res.items():
        ms = statistics.median(v)
        print(f"{k:28s} median {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s  (min {min(v):.3f} max {max(v):.3f})")


if __name__ == "__main__":
    main()
