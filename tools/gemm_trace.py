"""Per-CTA timeline of one GEMM launch (clock64 stamps recorded by the kernel when
rf_gemm_set_trace is set): main-loop time per tile, MMA waits on the accumulator, TMA
lead, epilogue time.  python tools/gemm_trace.py [N K epi]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native, tensor_ops as ops  # noqa: E402


def trace(M, N, K, epi, bn, pair, label, sk=False):
    lib = _native.load()
    lib.rf_gemm_set_trace.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(148 * 16 * 8, dtype=torch.int64, device="cuda")
    a = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    h = torch.randn(M, N, device="cuda")
    gate = torch.randn(4, N, device="cuda")
    kw = dict(out=h, epilogue=ops.EPI_RESID_GATE, gate=gate, rows_per_batch=750) if epi == "resid" else \
        dict(epilogue=ops.EPI_BF16)
    for _ in range(3):
        ops.gemm(a, w, block_n=bn, pair=pair, stream_k=sk, **kw)
    torch.cuda.synchronize()
    lib.rf_gemm_set_trace(buf.data_ptr())
    ops.gemm(a, w, block_n=bn, pair=pair, stream_k=sk, **kw)
    torch.cuda.synchronize()
    lib.rf_gemm_set_trace(None)
    t = buf.cpu().numpy().reshape(148, 16, 8).astype(np.float64)
    leaders = range(0, 148, 2) if pair else range(148)
    mains, waits, epis, leads, ntiles = [], [], [], [], []
    for c in leaders:
        n = int(np.sum(t[c, :, 0] > 0))
        ntiles.append(n)
        for i in range(n):
            mains.append(t[c, i, 3] - t[c, i, 2])         # first stage ready -> last MMA issued
            waits.append(t[c, i, 1] - t[c, i, 0])         # MMA waiting for a free accumulator
            leads.append(t[c, i, 2] - t[c, i, 1])         # accumulator free -> first stage ready
            if t[c, i, 5] > 0:
                epis.append(t[c, i, 5] - t[c, i, 4])      # epilogue (warp 2)
    span = [t[c, :, 5].max() - t[c, 0, 0] for c in leaders]
    if sk:   # per-segment timeline of a few units (cycles from the unit's first MMA wait)
        for c in (0, 2, 74, 146):
            n = int(np.sum(t[c, :, 0] > 0))
            b0 = t[c, 0, 0]
            segs = " | ".join(f"mma {t[c, i, 2] - b0:6.0f}-{t[c, i, 3] - b0:6.0f} epi {t[c, i, 4] - b0:6.0f}-{t[c, i, 5] - b0:6.0f}"
                              for i in range(n))
            print(f"   cta {c:3d}: {segs}")
    f = lambda v: f"{np.median(v):8.0f} (max {np.max(v):8.0f})" if len(v) else "-"
    ent, post, ext = t[:, 15, 7], t[:, 13, 7], t[:, 14, 7]
    print(f"{label}: globaltimer kernel span {(ext.max() - ent.min()) / 1e3:.1f} us; entry spread "
          f"{(ent.max() - ent.min()) / 1e3:.1f} us; entry->after pdl/prologue median {np.median(post - ent) / 1e3:.2f} us; "
          f"CTA duration median {np.median(ext - ent) / 1e3:.1f} us; cycles/us {np.median(span) / max(1e-9, np.median(ext - post) / 1e3):.0f}")
    print(f"{label}: tiles/unit {min(ntiles)}-{max(ntiles)} | mainloop cyc {f(mains)} | acc-wait {f(waits)} | "
          f"stage-lead {f(leads)} | epilogue {f(epis)} | span {f(span)}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "sk":
        for (N, K) in ((2048, 2048), (2048, 6144)):
            for epi in ("bf16", "resid"):
                for sk in (False, True):
                    trace(3000, N, K, epi, 128, True, f"N={N} K={K} {epi:5s} bn=128 pair=1 sk={int(sk)}", sk)
        sys.exit(0)
    for (N, K) in ((2048, 2048), (2048, 6144), (12288, 2048)):
        for epi in ("bf16", "resid"):
            for bn, pair in ((128, True), (256, True), (128, False)):
                trace(3000, N, K, epi, bn, pair, f"N={N} K={K} {epi:5s} bn={bn} pair={int(pair)}")
