"""Tensor-core decode vs the float64 kernel and the oracle, plus timings (GPU box).

python tools/decode_tc_check.py  -> prints LSB stats and per-shape timings.
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2605_28657_b200 as rf  # noqa: E402
import oracle.ringflow_np as O  # noqa: E402
import scenarios  # noqa: E402


def lsb(a, b):
    d = np.abs(a.astype(np.int32) - b.astype(np.int32))
    return int(d.max()) if d.size else 0, float(np.mean(d > 0)) if d.size else 0.0


def timeit(fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph, replayed (no host gaps)."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay()
        st.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            s.record(st)
            g.replay()
            e.record(st)
            st.synchronize()
            best = min(best, s.elapsed_time(e) / reps)
    return best


def main():
    for C, hop, T in ((8, 64, 96), (64, 1920, 300)):
        codec = rf.ToyCodec(channels=C, hop=hop)
        print(f"C={C} hop={hop}: tensor_cores={codec.tensor_cores}", flush=True)
        lat = scenarios.keyed(7, "tc-check", (T, C)) * 0.7
        tc_full = codec.full_decode(lat).samples
        ref = O.Codec(C, hop).full(lat)
        print("  full vs oracle (max lsb, frac differ):", lsb(tc_full, ref), flush=True)
        packed = codec._packed
        codec._packed = None
        f64_full = codec.full_decode(lat).samples
        codec._packed = packed
        print("  full vs f64 kernel:", lsb(tc_full, f64_full), " f64 vs oracle:", lsb(f64_full, ref), flush=True)
        ok = True
        rng = np.random.default_rng(0)
        for _ in range(20):
            a = int(rng.integers(0, T - 1))
            b = int(min(T, a + rng.integers(1, 200)))
            w = codec.windowed_decode(lat, (a, b), 15).samples
            ok &= np.array_equal(w, tc_full[a * hop:b * hop])
            r = O.Codec(C, hop).window(lat, a, b, 15)
            m, _ = lsb(w, r)
            ok &= m <= 1
        print("  windowed == full bit-exact and <=1 LSB vs oracle windows:", ok, flush=True)
    codec = rf.ToyCodec(channels=64, hop=1920)
    for T, (a, b), name in ((1500, (1425, 1500), "3-s window of 60 s"), (6000, (0, 6000), "240-s full")):
        lat = torch.from_numpy(scenarios.keyed(3, "tc-time", (T, 64)) * 0.7).cuda()
        out = torch.empty((b - a) * 1920, dtype=torch.int16, device="cuda")
        full = (a, b) == (0, T)
        ov = 0 if full else 15
        t_tc = timeit(lambda: codec.decode_device(lat, a, b, ov, full, out=out))
        packed = codec._packed
        codec._packed = None
        t_64 = timeit(lambda: codec.decode_device(lat, a, b, ov, full, out=out))
        codec._packed = packed
        print(f"{name}: tensor-core {t_tc * 1e3:.1f} us, float64 kernel {t_64 * 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
