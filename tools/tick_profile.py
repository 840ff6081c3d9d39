"""Host-side cost of StreamPipeline.tick() at config 2 with the DiT (cProfile, GPU box).
Prints the wall time per tick, the device time per tick, and the top host functions."""
import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
import paper_2605_28657_b200 as rf  # noqa: E402
from paper_2605_28657_b200 import dit as dit_mod  # noqa: E402


def main():
    conf = rf.PipelineConfig(depth=4, steps=8, frames=1500, channels=64, seed=0)
    if "--toy" in sys.argv:   # the reference's own velocity model
        pipe = rf.StreamPipeline(conf, request=bench.make_request(rf, 0))
    else:
        model = dit_mod.DiT(dit_mod.DiTConfig(), frames=1500, max_rows=4)
        pipe = rf.StreamPipeline(conf, request=bench.make_request(rf, 0), velocity_model=dit_mod.DiTVelocity(model))
    for _ in range(12):
        pipe.tick()
    torch.cuda.synchronize()
    n = 40
    t0 = time.perf_counter()
    host = 0.0
    for _ in range(n):
        h0 = time.perf_counter()
        pipe.tick()
        host += time.perf_counter() - h0
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e3
    print(f"wall {wall:.3f} ms/tick, host inside tick() {host / n * 1e3:.3f} ms/tick")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(n):
        pipe.tick()
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(30)


if __name__ == "__main__":
    main()
