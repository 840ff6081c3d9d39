"""DiT forward: accuracy vs the fp32 oracle and device time / TFLOP/s at config-2 shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402
from oracle.dit_fp32 import reference_forward  # noqa: E402


def main():
    # a non-default stream, so the forward runs as its captured CUDA graph
    torch.cuda.set_stream(torch.cuda.Stream())
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    frames = next((int(a.split("=")[1]) for a in sys.argv if a.startswith("--frames=")), 1500)
    cfg = D.DiTConfig()
    dit = D.DiT(cfg, frames=frames, max_rows=max(rows, 8))
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(frames, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(rows)]
    ts = [1.0 - 0.1 * i for i in range(rows)]
    conds = [dit.cond_tokens(i) for i in range(rows)]
    out = dit.forward(xs, ts, conds).clone()
    if "--no-ref" not in sys.argv:
        ref = reference_forward(dit, xs, ts, conds)
        err = ((out - ref).pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()).item()
        print(f"rows={rows} rel_rms_vs_fp32={err:.3e} out_rms={out.pow(2).mean().sqrt().item():.3f}")
    for _ in range(3):
        dit.forward(xs, ts, conds)
    torch.cuda.synchronize()
    n = 10
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        dit.forward(xs, ts, conds)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    fl = cfg.flops_per_forward(rows, frames)
    print(f"forward {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s  ({fl / 1e12:.2f} TFLOP)  params={cfg.params() / 1e9:.2f}B")
    if "--graph" in sys.argv:   # same forward replayed from a CUDA graph (no host launch gaps)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            dit.forward(xs, ts, conds)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                dit.forward(xs, ts, conds)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(n):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        gms = a.elapsed_time(b) / n
        print(f"graph forward {gms:.3f} ms  {fl / gms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
