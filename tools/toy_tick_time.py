"""Device time per config-2 toy tick (bench.timed_ticks: events on the pipeline stream around
each tick, L2 flushed before each) -- the toy_path leg of bench.py alone.  python tools/toy_tick_time.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_28657_b200 as rf  # noqa: E402

conf = rf.PipelineConfig(depth=bench.DEPTH, steps=bench.STEPS, frames=bench.T, channels=bench.D, seed=0)
p = rf.StreamPipeline(conf, request=bench.make_request(rf, 0))
for _ in range(32):
    p.tick()
torch.cuda.synchronize()
flush = torch.empty(bench.L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
res = []
for _ in range(3):
    ms, done, launches = bench.timed_ticks(p, 64, flush, p.stream)
    res.append(ms / 64 * 1e3)
print("toy tick device us:", " ".join(f"{x:.2f}" for x in res), f" ({launches / 64:.1f} launches per tick)")
