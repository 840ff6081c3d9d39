"""bench.py's timed-tick loop, with the per-tick device times split by whether the PREVIOUS
tick completed a generation (its host sync can leave the GPU idle at the start of the next
tick) -- and the model-phase time of the same ticks."""
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
        evs, prev_done = [], []
        last = 0
        for _ in range(24):
            if use_flush:
                with torch.cuda.stream(st):
                    flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            n = len(pipe.tick())
            b.record(st)
            evs.append((a, b))
            prev_done.append(last)
            last = n
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) for a, b in evs]
        after = [t for t, p in zip(ts, prev_done) if p]
        other = [t for t, p in zip(ts, prev_done) if not p]
        print(f"flush={use_flush}: all {sum(ts) / len(ts):.3f} ms | after a completing tick {sum(after) / max(1, len(after)):.3f} "
              f"(n={len(after)}) | otherwise {sum(other) / max(1, len(other)):.3f} (n={len(other)})")


if __name__ == "__main__":
    main()
