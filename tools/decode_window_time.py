"""3-s window decode (75 frames + 15 overlap, C=64, hop 1920) device time, three ways:
back-to-back launches (device time per launch), one launch behind a busy stream (what the
bench's events see when the host enqueues faster than the GPU drains), and one launch on an
idle stream (includes the host's enqueue latency)."""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2605_28657_b200 as rf  # noqa: E402
import scenarios  # noqa: E402

T, W, OV = 1500, 75, 15
codec = rf.ToyCodec(channels=64, hop=1920)
lat = torch.from_numpy(scenarios.keyed(3, "tc-time", (T, 64)) * 0.7).cuda()
out = torch.empty(W * 1920, dtype=torch.int16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    codec.decode_device(lat, T - W, T, OV, False, out=out)
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
a, b = E(), E()
a.record()
for _ in range(100):
    codec.decode_device(lat, T - W, T, OV, False, out=out)
b.record()
torch.cuda.synchronize()
print(f"back-to-back: {a.elapsed_time(b) / 100 * 1e3:.2f} us per window")
for label, mode in (("behind flush (dirty L2)", "dirty"), ("behind flush + read-back (clean L2)", "clean"),
                    ("idle stream", "idle")):
    res = []
    for _ in range(20):
        if mode == "idle":
            torch.cuda.synchronize()
        else:
            flush.fill_(1)
            if mode == "clean":
                torch.amax(flush)
        a, b = E(), E()
        a.record()
        codec.decode_device(lat, T - W, T, OV, False, out=out)
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) * 1e3)
    print(f"{label}: median {statistics.median(res):.2f} us (min {min(res):.2f})")
