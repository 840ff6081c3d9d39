"""In-graph cost of each DiT kernel class: the config-2 forward (4 rows) timed as a CUDA
graph with one class left out at a time (RF_DIT_SKIP, read once per process, so every
variant runs in its own subprocess); cost = full - ablated.  Timing only."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLASSES = [("norms x3", 1), ("self-attn", 2), ("cross-attn", 4), ("QKV gemm", 8), ("O gemm", 16),
           ("cross-Q gemm", 32), ("cross-O gemm", 64), ("gate-up gemm", 128), ("down gemm", 256)]
CHILD = r'''
import os, sys, torch
sys.path.insert(0, %r)
from paper_2605_28657_b200 import dit as D
torch.cuda.set_stream(torch.cuda.Stream())
cfg = D.DiTConfig()
dit = D.DiT(cfg, frames=1500, max_rows=4)
g = torch.Generator(device="cuda").manual_seed(0)
xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(4)]
ts = [1.0 - 0.1 * i for i in range(4)]
conds = [dit.cond_tokens(i) for i in range(4)]
for _ in range(5):
    dit.forward(xs, ts, conds)
torch.cuda.synchronize()
import subprocess as sp, tempfile
f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
mon = sp.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "50"],
               stdout=f, stderr=sp.DEVNULL)
best = []
for rep in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        dit.forward(xs, ts, conds)
    b.record()
    torch.cuda.synchronize()
    best.append(a.elapsed_time(b) / 5)
mon.terminate(); mon.wait(); f.flush()
vals = [l.split(",") for l in open(f.name).read().split("\n") if "," in l]
clk = sorted(float(v[0]) for v in vals); pw = sorted(float(v[1]) for v in vals)
print(f"CLK {clk[len(clk)//2]:.0f} PW {pw[len(pw)//2]:.0f}")
print(sorted(best)[len(best) // 2])
''' % ROOT


INFO = {}


def run(mask):
    env = dict(os.environ, RF_DIT_SKIP=str(mask))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    lines = out.stdout.strip().splitlines()
    if len(lines) < 2:
        raise RuntimeError(out.stderr[-2000:])
    INFO.setdefault(mask, []).append(lines[-2])
    return float(lines[-1])


def masks(ms):
    for m in ms:
        ts = [run(m) for _ in range(3)]
        print(f"RF_DIT_SKIP={m:4d}: {sorted(ts)[1]:.3f} ms  {INFO[m][0]}", flush=True)


def main():
    if len(sys.argv) > 1:
        return masks([int(x) for x in sys.argv[1:]])
    full = [run(0)]
    res = []
    for name, m in CLASSES:
        res.append((name, run(m)))
        full.append(run(0))
    f = sorted(full)[len(full) // 2]
    print(f"full forward {f:.3f} ms (runs: {' '.join(f'{x:.3f}' for x in full)})")
    for name, t in res:
        print(f"  {name:14s} {f - t:7.3f} ms per forward ({(f - t) / 24 * 1e3:6.1f} us per layer)  [{t:.3f}]  "
              f"{INFO[dict(CLASSES)[name]][0]}")
    print("full:", INFO[0])


if __name__ == "__main__":
    main()
