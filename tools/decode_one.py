"""Run one decode shape a few times (for ncu captures):  python tools/decode_one.py T a b [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2605_28657_b200 as rf  # noqa: E402
import scenarios  # noqa: E402

T, a, b = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 6
codec = rf.ToyCodec(channels=64, hop=1920)
lat = torch.from_numpy(scenarios.keyed(3, "tc-time", (T, 64)) * 0.7).cuda()
out = torch.empty((b - a) * 1920, dtype=torch.int16, device="cuda")
full = (a, b) == (0, T)
for _ in range(reps):
    codec.decode_device(lat, a, b, 0 if full else 15, full, out=out)
torch.cuda.synchronize()
