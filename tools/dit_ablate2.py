"""In-situ cost of DiT kernel classes with VALID data: one DiT runs full forwards first (all
buffers hold real activations), then rf_dit_set_skip leaves a class out (the skipped kernels'
outputs stay as the last full forward left them, so downstream kernels see realistic data);
masks alternate round by round.  cost = full - ablated.

    python tools/dit_ablate2.py [mask ...]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native, dit as D  # noqa: E402

NAMES = {0: "full", 1: "norms x3", 2: "self-attn", 4: "cross-attn", 8: "QKV", 16: "O", 32: "cross-Q",
         64: "cross-O", 128: "gate-up", 256: "down", 3: "norms+self-attn", 7: "norms+attn", 510: "norms only",
         509: "self-attn only", 507: "cross-attn only", 511: "nothing per-layer"}


def main():
    masks = [int(x) for x in sys.argv[1:]] or [0, 1, 2, 4, 8, 16, 32, 64, 128, 256, 7, 511]
    lib = _native.load()
    lib.rf_dit_set_skip.argtypes = [ctypes.c_void_p, ctypes.c_int32]
    torch.cuda.set_stream(torch.cuda.Stream())
    dit = D.DiT(D.DiTConfig(), frames=1500, max_rows=4)
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(4)]
    ts = [1.0 - 0.1 * i for i in range(4)]
    conds = [dit.cond_tokens(i) for i in range(4)]
    for _ in range(3):
        dit.forward(xs, ts, conds)
    res = {m: [] for m in masks}
    for _ in range(6):
        for m in masks:
            lib.rf_dit_set_skip(dit.handle, m)
            for _ in range(2):
                dit.forward(xs, ts, conds)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(4):
                dit.forward(xs, ts, conds)
            b.record()
            torch.cuda.synchronize()
            res[m].append(a.elapsed_time(b) / 4)
    lib.rf_dit_set_skip(dit.handle, 0)
    med = {m: sorted(v)[len(v) // 2] for m, v in res.items()}
    full = med.get(0)
    for m in masks:
        extra = f"  cost {full - med[m]:6.3f} ms ({(full - med[m]) / 24 * 1e3:6.1f} us/layer)" if full and m else ""
        print(f"{NAMES.get(m, m)!s:18s} mask {m:4d}: {med[m]:7.3f} ms{extra}", flush=True)


if __name__ == "__main__":
    main()
