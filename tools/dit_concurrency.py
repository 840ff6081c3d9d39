"""DiT forwards on one stream while another stream keeps the GPU busy with library kernels
(cuBLAS fp32 GEMMs), as the trajectory tests do with the oracle: every forward must finish."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402


def main():
    s_dit, s_other = torch.cuda.Stream(), torch.cuda.Stream()
    dit = D.DiT(D.DiTConfig(), frames=1500, max_rows=8)
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(8)]
    conds = [dit.cond_tokens(i) for i in range(8)]
    a = torch.randn(3000, 2048, device="cuda")
    w = torch.randn(2048, 2048, device="cuda")
    torch.cuda.synchronize()
    for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
        rows = 1 + it % 8
        with torch.cuda.stream(s_other):
            for _ in range(200):
                a = torch.tanh(a @ w * 1e-3)
        with torch.cuda.stream(s_dit):
            dit.forward(xs[:rows], [1.0 - 0.1 * i for i in range(rows)], conds[:rows])
        t0 = time.time()
        s_dit.synchronize()
        print(f"iter {it} rows={rows} dit done in {time.time() - t0:.3f} s", flush=True)
        s_other.synchronize()


if __name__ == "__main__":
    main()
