"""Generate golden vectors by running the REAL reference in the build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_goldens.py

/root/reference exists only in the build container (not on the GPU box), so its
outputs are frozen here as small fixtures.  Written with numpy 2.3.5 / Python 3.12.3.
Large arrays are stored as sha256 digests of their float64 / int16 bytes (a bit-exact
check), small ones in full.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))          # tests/
sys.path.insert(0, "/root/reference/pkg/src")

import ringflow  # noqa: E402  (the reference)
from ringflow.codec import quantize_pcm  # noqa: E402

import scenarios  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def noise_goldens(out):
    cases = [(0, 0, 0, "sde", 4), (7, 12345, 3, "model", 1000), (2**40, -99, 7, "init", 96000),
             (3, 2**62, 1, "decoder-conv", 3 * 64 * 64), (11, 5, 0, "amps", 1), (0, 0, 0, "x", 0)]
    for i, (seed, stream, step, tag, n) in enumerate(cases):
        ns = ringflow.NoiseSource(seed=seed, stream=stream)
        v = ns.normal(step, tag, (n,))
        u = ns.uniform(step, tag, (n,))
        out[f"noise{i}_args"] = np.array([seed, stream, step, n], dtype=object)
        out[f"noise{i}_tag"] = np.array(tag)
        out[f"noise{i}_normal_sha"] = np.array(digest(v))
        out[f"noise{i}_uniform_sha"] = np.array(digest(u))
        out[f"noise{i}_normal_head"] = v[:64].copy()
    # a long draw: ~1e6 normals exercise thousands of wedge and ~100 tail events
    ns = ringflow.NoiseSource(seed=123, stream=456)
    out["noise_long_sha"] = np.array(digest(ns.normal(9, "long", (1_000_000,))))


def schedule_goldens(out):
    rows = []
    for d in (1.0, 0.5, 0.7, 0.25, 1e-3):
        for s in (1, 4, 8, 13):
            for sh in (3.0, 1.0):
                sc = ringflow.build_schedule(d, s, sh)
                rows.append((d, s, sh, sc.schedule_id, digest(sc.sigmas)))
    out["sched_rows"] = np.array(rows, dtype=object)


def codec_goldens(out):
    lat = ringflow.NoiseSource(seed=300).normal(0, "codec-fixture", (96, 8))
    codec = ringflow.ToyCodec(channels=8, hop=64)
    out["codec8_latent"] = lat
    out["codec8_full"] = codec.full_decode(lat).samples
    rng = np.random.default_rng(5)
    wins = []
    for _ in range(12):
        a = int(rng.integers(0, 95))
        b = int(rng.integers(a + 1, 97))
        for ov in (15, 0, 3):
            ch = codec.windowed_decode(lat, (a, b), ov)
            wins.append((a, b, ov, codec.frames_decoded_last))
            out[f"codec8_win_{a}_{b}_{ov}"] = ch.samples
    out["codec8_windows"] = np.array(wins, dtype=np.int64)
    out["codec8_rf"] = np.array(ringflow.measure_receptive_field(codec))
    # ACE-Step-shape latent channels and 48 kHz hop: C=64, hop=1920
    lat64 = ringflow.NoiseSource(seed=301).normal(0, "codec-fixture", (40, 64))
    codec64 = ringflow.ToyCodec(channels=64, hop=1920)
    out["codec64_latent"] = lat64
    out["codec64_full"] = codec64.full_decode(lat64).samples
    out["codec64_win"] = codec64.windowed_decode(lat64, (10, 25), 15).samples
    q = quantize_pcm(np.array([0.0, 0.5 / 32767, -0.5 / 32767, 1.0, -1.0, 2.0, -2.0]))
    out["quantize_kat"] = q


def scenario_goldens(out):
    for name, spec in scenarios.SPECS.items():
        tr = scenarios.drive(ringflow, spec)
        for k, v in tr.items():
            if k == "latents":
                out[f"sc_{name}_latent_sha"] = np.array([digest(x) for x in v]) if len(v) else np.zeros(0, "U64")
                if len(v):
                    out[f"sc_{name}_latent_last"] = v[-1]
            else:
                out[f"sc_{name}_{k}"] = v


def main():
    out = {}
    noise_goldens(out)
    schedule_goldens(out)
    codec_goldens(out)
    scenario_goldens(out)
    out["numpy_version"] = np.array(np.__version__)
    path = os.path.join(HERE, "reference_goldens.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
