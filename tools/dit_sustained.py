"""Sustained DiT forward rate: 2 s of back-to-back graph replays (config 2, 4 rows) after a
1 s warm-up, median over 20 groups of 10 -- the board-power-capped steady state the tick runs
in (short runs read a few % faster on a cool GPU)."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402


def main():
    torch.cuda.set_stream(torch.cuda.Stream())
    cfg = D.DiTConfig()
    dit = D.DiT(cfg, frames=1500, max_rows=4)
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(4)]
    ts = [1.0 - 0.1 * i for i in range(4)]
    conds = [dit.cond_tokens(i) for i in range(4)]
    t0 = time.time()
    while time.time() - t0 < 1.0:
        dit.forward(xs, ts, conds)
    torch.cuda.synchronize()
    res = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            dit.forward(xs, ts, conds)
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 10)
    ms = statistics.median(res)
    print(f"sustained forward {ms:.3f} ms  {cfg.flops_per_forward(4, 1500) / ms / 1e9:.1f} TFLOP/s "
          f"(min {min(res):.3f} max {max(res):.3f})")


if __name__ == "__main__":
    main()
