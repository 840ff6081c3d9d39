"""Timeline of the tensor-core window decode (3-s window + 15 overlap, C=64, hop 1920): the
kernel's globaltimer stamps (rf_decode_set_trace) of every CTA, relative to the first CTA's
entry, after warm-up.  python tools/decode_trace.py [start stop]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2605_28657_b200 as rf  # noqa: E402
import scenarios  # noqa: E402
from paper_2605_28657_b200 import _native  # noqa: E402

T = 1500
a, b = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (T - 75, T)
codec = rf.ToyCodec(channels=64, hop=1920)
lat = torch.from_numpy(scenarios.keyed(3, "tc-time", (T, 64)) * 0.7).cuda()
out = torch.empty((b - a) * 1920, dtype=torch.int16, device="cuda")
lib = _native.load()
buf = torch.zeros(4096 * 32, dtype=torch.int64, device="cuda")
NAMES = {0: "entry", 1: "tmem+sync", 17: "latent written", 12: "ups operand rdy", 31: "exit"}
for l in range(4):
    NAMES[2 + 2 * l] = f"L{l} operand rdy"
    NAMES[3 + 2 * l] = f"L{l} weights rdy"
    NAMES[18 + l] = f"L{l} acc rdy"
for j in range(4):
    NAMES[13 + j] = f"chunk{j} weights rdy"
for it in range(6):
    lib.rf_decode_set_trace(ctypes.c_void_p(buf.data_ptr() if it == 5 else 0))
    buf.zero_()
    codec.decode_device(lat, a, b, 15, False, out=out)
    torch.cuda.synchronize()
lib.rf_decode_set_trace(ctypes.c_void_p(0))
t = buf.view(4096, 32).cpu().numpy()
ctas = [i for i in range(4096) if t[i, 0] > 0]
t0 = min(t[i, 0] for i in ctas)
print(f"{len(ctas)} CTAs; times in us from the first entry")
for s in sorted(NAMES, key=lambda k: [0, 1, 17, 2, 3, 18, 4, 5, 19, 6, 7, 20, 8, 9, 21, 12, 13, 14, 15, 16, 31].index(k)):
    v = [(t[i, s] - t0) / 1e3 for i in ctas if 0 < t[i, s] < 2 ** 62]
    if v:
        print(f"{NAMES[s]:18s} min {min(v):7.2f}  max {max(v):7.2f}")
