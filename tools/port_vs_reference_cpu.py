"""Build-container check that the oracle port costs what the real reference costs on CPU.

    PYTHONPATH=/root/reference/pkg/src python tools/port_vs_reference_cpu.py
Times config-2-shape ticks (T=1500, D=64, depth 4, S=8, toy model) of the real reference
StreamPipeline and of oracle/ringflow_np.py, single thread.  (The reference cannot travel
to the GPU box, so the bench's CPU arm runs the port; this shows it is a faithful stand-in.)
"""
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import ringflow  # noqa: E402
import scenarios  # noqa: E402

import oracle.ringflow_np as O  # noqa: E402

T, D = 1500, 64


def rate(tick, warm=32, seconds=8.0):
    for _ in range(warm):
        tick()
    n, done, t0 = 0, 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        done += len(tick())
        n += 1
    dt = time.perf_counter() - t0
    return done / dt, dt / n * 1e3


src = scenarios.keyed(0, "bench-source", (T, D))
ref = ringflow.StreamPipeline(ringflow.PipelineConfig(depth=4, steps=8, frames=T, channels=D),
                              request=ringflow.GenerationRequest(conditions=(ringflow.ConditionSet(
                                  ringflow.content_hash("bench", "bench prompt"), source=src),)))
port = O.Pipeline(depth=4, steps=8, frames=T, channels=D,
                  request=O.Request([O.Cond(O.chash("bench", "bench prompt"), source=src)]))
r = rate(ref.tick)
p = rate(port.tick)
print(f"reference: {r[0]:.2f} completions/s ({r[1]:.2f} ms/tick); port: {p[0]:.2f} completions/s "
      f"({p[1]:.2f} ms/tick); port/reference = {p[0] / r[0]:.3f}")
