"""Host time per tick section of the toy path (perf_counter wrappers around the pipeline's
methods), config-2 shape.  python tools/toy_host_sections.py [ticks]"""
import collections
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
import paper_2605_28657_b200 as rf  # noqa: E402
from paper_2605_28657_b200 import pipeline as P  # noqa: E402

acc = collections.defaultdict(float)


def wrap(cls, name):
    fn = getattr(cls, name)

    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            acc[name] += time.perf_counter() - t
    setattr(cls, name, w)


for n in ("tick", "_tick_begin", "_step_slots", "_tick_end", "_emit_launch", "_emit_finish", "_refill",
          "_init_slots", "_curve_view"):
    wrap(P.StreamPipeline, n)
from paper_2605_28657_b200 import _native  # noqa: E402
_lib = _native.load()
for _name in ("rf_tick_solve", "rf_emit_stats", "rf_admit_init"):
    _f = getattr(_lib, _name)

    def _w(*a, _f=_f, _name=_name):
        t = time.perf_counter()
        try:
            return _f(*a)
        finally:
            acc["C:" + _name] += time.perf_counter() - t
    setattr(_lib, _name, _w)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    conf = rf.PipelineConfig(depth=4, steps=8, frames=1500, channels=64, seed=0)
    pipe = rf.StreamPipeline(conf, request=bench.make_request(rf, 0))
    for _ in range(64):
        pipe.tick()
    torch.cuda.synchronize()
    acc.clear()
    t0 = time.perf_counter()
    for _ in range(n):
        pipe.tick()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e6
    print(f"wall {wall:.1f} us/tick")
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
        print(f"  {k:14s} {v / n * 1e6:7.1f} us/tick")


if __name__ == "__main__":
    main()
