"""Forward the full-size DiT at every row count 1..max_rows (one process; prints as it goes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402


def main():
    torch.cuda.set_stream(torch.cuda.Stream())
    mr = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
    dit = D.DiT(D.DiTConfig(), frames=frames, max_rows=mr)
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(frames, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(mr)]
    conds = [dit.cond_tokens(i) for i in range(mr)]
    order = [int(a) for a in sys.argv[3].split(",")] if len(sys.argv) > 3 else list(range(1, mr + 1))
    for rows in order:
        for rep in range(3):
            out = dit.forward(xs[:rows], [1.0 - 0.1 * i for i in range(rows)], conds[:rows])
            torch.cuda.synchronize()
        print(f"rows={rows} ok finite={bool(torch.isfinite(out[:rows]).all())}", flush=True)


if __name__ == "__main__":
    main()
