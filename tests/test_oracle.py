"""Pin the CPU oracle against golden vectors produced by the real reference (CPU only)."""
import ctypes
import hashlib
import os
import subprocess

import numpy as np
import pytest

import oracle.ringflow_np as O
import scenarios

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def clib():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_build", "liboracle_npyrandom.so"))
    lib.oracle_normal_fill.restype = ctypes.c_uint64
    lib.oracle_normal_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
    lib.oracle_uniform_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
    return lib


def c_normal(lib, key, n):
    out = np.empty(n)
    lib.oracle_normal_fill(key & (2**64 - 1), key >> 64, n, out.ctypes.data)
    return out


def test_noise_kat_survey():
    # NoiseSource(0,0).normal(0,"sde",(4,))
    v = O.normal(0, 0, 0, "sde", (4,))
    assert v.tolist() == [-0.8766545588837262, 1.8638264440516052, -0.3612334156474177, -1.833676777774578]


def test_noise_goldens(goldens):
    for i in range(6):
        seed, stream, step, n = goldens[f"noise{i}_args"]
        tag = str(goldens[f"noise{i}_tag"])
        assert sha(O.normal(seed, stream, step, tag, (n,))) == str(goldens[f"noise{i}_normal_sha"])
        assert sha(O.uniform(seed, stream, step, tag, (n,))) == str(goldens[f"noise{i}_uniform_sha"])


def test_c_restatement_matches_golden(goldens, clib):
    """oracle/npyrandom.c (the algorithm the GPU implements) == the reference's numpy stream."""
    for i in range(6):
        seed, stream, step, n = goldens[f"noise{i}_args"]
        tag = str(goldens[f"noise{i}_tag"])
        key = O.philox_key(int(seed), int(stream), int(step), tag)
        assert sha(c_normal(clib, key, int(n))) == str(goldens[f"noise{i}_normal_sha"])
    key = O.philox_key(123, 456, 9, "long")
    assert sha(c_normal(clib, key, 1_000_000)) == str(goldens["noise_long_sha"])


def test_c_restatement_many_keys(clib):
    rng = np.random.default_rng(0)
    for _ in range(20):
        key = int(rng.integers(0, 2**63)) << 64 | int(rng.integers(0, 2**63))
        n = int(rng.integers(1, 50_000))
        ref = np.random.Generator(np.random.Philox(key=key)).standard_normal(n)
        assert np.array_equal(ref.view(np.uint64), c_normal(clib, key, n).view(np.uint64))


def test_schedule_goldens(goldens):
    for d, s, sh, sid, dg in goldens["sched_rows"]:
        sig = O.sigmas_of(d, s, sh)
        assert O.schedule_id(sig, sh) == sid
        assert sha(sig) == dg


def test_schedule_kats():
    assert O.schedule_id(O.sigmas_of(1.0, 8, 3.0), 3.0) == "9569fae88672"
    assert O.schedule_id(O.sigmas_of(0.5, 8, 3.0), 3.0) == "fe08daa1f91b"
    assert O.sigmas_of(1.0, 4, 3.0).tolist() == [1.0, 0.9, 0.75, 0.5, 0.0]


@pytest.mark.parametrize("name", sorted(scenarios.SPECS))
def test_oracle_scenarios_bit_exact(goldens, name):
    tr = scenarios.drive_oracle(scenarios.SPECS[name])
    for k in scenarios.EXACT_FIELDS:
        assert np.array_equal(tr[k], goldens[f"sc_{name}_{k}"]), k
    assert np.array_equal(np.array([sha(x) for x in tr["latents"]]), goldens[f"sc_{name}_latent_sha"])
    assert np.array_equal(np.nan_to_num(tr["rms"], nan=-1.0), np.nan_to_num(goldens[f"sc_{name}_rms"], nan=-1.0))


def test_codec_goldens(goldens):
    lat = goldens["codec8_latent"]
    codec = O.Codec(8, 64)
    assert np.array_equal(codec.full(lat), goldens["codec8_full"])
    for a, b, ov, _ in goldens["codec8_windows"]:
        assert np.array_equal(codec.window(lat, int(a), int(b), int(ov)), goldens[f"codec8_win_{a}_{b}_{ov}"])
    c64 = O.Codec(64, 1920)
    assert np.array_equal(c64.full(goldens["codec64_latent"]), goldens["codec64_full"])
    assert np.array_equal(c64.window(goldens["codec64_latent"], 10, 25, 15), goldens["codec64_win"])
    assert O.quantize(np.array([0.0, 0.5 / 32767, -0.5 / 32767, 1.0, -1.0, 2.0, -2.0])).tolist() == \
        goldens["quantize_kat"].tolist()


def test_cpu_dit_velocity_small_config():
    """oracle/dit_fp32.py (the fp32 DiT the CPU arm and the GPU parity tests use): a row's
    velocity matches its single-row forward up to bf16 rounding-point flips (the fp32 GEMMs
    differ in the last bits between batch shapes), and the model plugs into the oracle
    pipeline's model slot (finite velocities, the ring steps)."""
    import numpy as np
    import torch

    import oracle.ringflow_np as O
    from oracle.dit_fp32 import CpuDiTVelocity, forward_fp32
    from paper_2605_28657_b200.dit import DiTConfig

    cfg = DiTConfig().small()
    m = CpuDiTVelocity(cfg, frames=64, seed=3)
    g = torch.Generator().manual_seed(0)
    xs = [torch.randn(64, cfg.latent_channels, generator=g, dtype=torch.float64) for _ in range(3)]
    conds = [m.cond_tokens(i) for i in range(3)]
    with torch.no_grad():
        both = forward_fp32(cfg, m.W, 64, xs, [0.9, 0.5, 0.2], conds, f=lambda w: w)
        one = forward_fp32(cfg, m.W, 64, xs[1:2], [0.5], conds[1:2], f=lambda w: w)
    rel = ((both[1] - one[0]).pow(2).mean().sqrt() / one[0].pow(2).mean().sqrt()).item()
    assert rel < 1e-2, rel
    req = O.Request([O.Cond(O.chash("p", "x"), source=np.zeros((64, cfg.latent_channels)))])
    pipe = O.Pipeline(depth=2, steps=4, frames=64, channels=cfg.latent_channels, seed=0, request=req)
    pipe.model = m
    recs = []
    for _ in range(8):
        recs += pipe.tick()
    assert recs and all(np.isfinite(r.latent).all() for r in recs)
    # the bf16-operand CPU path (the CPU timing arm) stays within bf16 rounding of the fp32 one
    mb = CpuDiTVelocity(cfg, frames=64, seed=3, bf16=True)
    with torch.no_grad():
        vb = forward_fp32(cfg, mb.W, 64, xs[1:2], [0.5], conds[1:2], f=lambda w: w, bf16_matmul=True)
    rel = ((vb[0] - one[0]).pow(2).mean().sqrt() / one[0].pow(2).mean().sqrt()).item()
    assert rel < 3e-2, rel
