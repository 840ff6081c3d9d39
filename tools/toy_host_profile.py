"""Toy-path tick (config-2 shape, the reference's own model): wall-clock per tick, device
time per tick (events around the tick on the pipeline stream), and a cProfile of the host.

    python tools/toy_host_profile.py [ticks] [--no-cache]"""
import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
import paper_2605_28657_b200 as rf  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 400
    cache = "--no-cache" not in sys.argv
    conf = rf.PipelineConfig(depth=4, steps=8, frames=1500, channels=64, seed=0)
    pipe = rf.StreamPipeline(conf, request=bench.make_request(rf, 0), noise_cache_bytes=(256 << 20) if cache else 0)
    for _ in range(64):
        pipe.tick()
    torch.cuda.synchronize()
    st = pipe.stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    t0 = time.perf_counter()
    done = 0
    for i in range(n):
        evs[i][0].record(st)
        done += len(pipe.tick())
        evs[i][1].record(st)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e6
    dev = sum(a.elapsed_time(b) for a, b in evs) / n * 1e3
    print(f"cache={cache}: wall {wall:.1f} us/tick, device (tick-bracketed) {dev:.1f} us/tick, "
          f"{done / (wall * n / 1e6):.0f} completions/s wall")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        pipe.tick()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(22)


if __name__ == "__main__":
    main()
