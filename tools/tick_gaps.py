"""Where the device time of a tick goes: events at tick start/end plus the pipeline's phase
events, all on the pipeline stream; prints per-tick total, the phases, and the idle gaps
between consecutive events (device time not covered by any phase)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
import paper_2605_28657_b200 as rf  # noqa: E402
from paper_2605_28657_b200 import dit as dit_mod  # noqa: E402


def main():
    conf = rf.PipelineConfig(depth=4, steps=8, frames=1500, channels=64, seed=0)
    model = dit_mod.DiT(dit_mod.DiTConfig(), frames=1500, max_rows=4)
    pipe = rf.StreamPipeline(conf, request=bench.make_request(rf, 0), velocity_model=dit_mod.DiTVelocity(model))
    st = pipe.stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(12):
        pipe.tick()
    torch.cuda.synchronize()
    for use_flush in (True, False):
        phases = pipe.enable_phase_timing(True)
        ticks = []
        for _ in range(8):
            if use_flush:
                with torch.cuda.stream(st):
                    flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            n = len(pipe.tick())
            b.record(st)
            ticks.append((a, b, n))
        torch.cuda.synchronize()
        evs = [(name, s, e) for name, lst in phases.items() for s, e in lst]
        for a, b, n in ticks:
            inside = sorted([(a.elapsed_time(s), a.elapsed_time(e), name) for name, s, e in evs
                             if 0 <= a.elapsed_time(s) and b.elapsed_time(e) <= 0], key=lambda x: x[0])
            total = a.elapsed_time(b)
            parts, cur = [], 0.0
            for s0, e0, name in inside:
                parts.append(f"gap {s0 - cur:.3f} | {name} {e0 - s0:.3f}")
                cur = e0
            parts.append(f"gap {total - cur:.3f}")
            print(f"flush={int(use_flush)} emit={n} total {total:.3f} ms: " + " | ".join(parts), flush=True)
        pipe.enable_phase_timing(False)


if __name__ == "__main__":
    main()
