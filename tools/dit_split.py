"""Experiment: the 4-row DiT forward split into row groups on concurrent streams (shared
weights, one workspace per group) vs one batched forward.  Prints device ms per tick."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402


def run(groups, rows=4, n=10):
    cfg = D.DiTConfig()
    base = D.DiT(cfg, frames=1500, max_rows=max(groups))
    dits = [base] + [D.DiT(cfg, frames=1500, max_rows=max(groups), weights=base.weights) for _ in groups[1:]]
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(rows)]
    ts = [1.0 - 0.1 * i for i in range(rows)]
    conds = [base.cond_tokens(i) for i in range(rows)]
    streams = [torch.cuda.Stream() for _ in groups]
    ref = base.forward(xs, ts, conds).clone() if len(groups) == 1 else None

    def tick():
        main = torch.cuda.current_stream()
        i = 0
        for d, s, k in zip(dits, streams, groups):
            s.wait_stream(main)
            with torch.cuda.stream(s):
                d.forward(xs[i:i + k], ts[i:i + k], conds[i:i + k])
            i += k
        for s in streams:
            main.wait_stream(s)

    for _ in range(3):
        tick()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        tick()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    print(f"groups={groups}: {ms:.3f} ms/tick  {cfg.flops_per_forward(rows, 1500) / ms / 1e9:.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    for gr in ([4], [2, 2], [1, 1, 1, 1], [3, 1]):
        run(gr)
