"""Run config-2-shape ticks of the toy-velocity pipeline (the reference's own model) --
a driver for profiling the per-tick kernels (rf_tick_kernel, noise, emit, admit) under ncu.

    python tools/toy_ticks.py [ticks]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
import paper_2605_28657_b200 as rf  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    conf = rf.PipelineConfig(depth=4, steps=8, frames=1500, channels=64, seed=0)
    pipe = rf.StreamPipeline(conf, request=bench.make_request(rf, 0))
    done = 0
    for _ in range(n):
        done += len(pipe.tick())
    torch.cuda.synchronize()
    print(f"{n} ticks, {done} completions")


if __name__ == "__main__":
    main()
