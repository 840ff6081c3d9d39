"""Toy-path device time per tick and per phase (bench.timed_ticks), config-2 shape."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
import paper_2605_28657_b200 as rf  # noqa: E402

conf = rf.PipelineConfig(depth=4, steps=8, frames=1500, channels=64, seed=0)
tp = rf.StreamPipeline(conf, request=bench.make_request(rf, 0))
for _ in range(40):
    tp.tick()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(2):
    ms, done, _ = bench.timed_ticks(tp, 64, flush, tp.stream)
    ph = bench.timed_ticks(tp, 32, flush, tp.stream, phases=True)[3]
    print(f"{ms / 64 * 1e3:.1f} us/tick, phases " + ", ".join(f"{k} {v * 1e3:.1f}" for k, v in ph.items()))
