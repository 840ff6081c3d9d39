"""Trajectory-level DiT parity: the bf16 GPU ring vs the reference tick with a TRUE fp32 DiT.

``north_star``: outputs "within a stated bf16-vs-fp32 tolerance on latents and audio after the
full S-step trajectory".  Both sides run the same ring at config-2 shape (ACE-Step-shape
24-layer DiT, T=1500, D=64, depth 4, S=8) on the same seeded weights, conditioning tokens
and keyed noise (the noise is bit-exact, tests/test_gpu_noise.py), so every difference is
the DiT's arithmetic:

* GPU: ``StreamPipeline`` + ``DiTVelocity`` -- bf16 GEMM / attention operands, fp32
  accumulation and fp32 residual stream (csrc/rf_dit.cu), float64 ring and solver.
* oracle: ``oracle/ringflow_np.Pipeline`` (the reference tick restated,
  reference pipeline.py:424-464 / solver.py:141-306) with ``Fp32DiTVelocity`` in its model
  slot -- the same network with NO bf16 rounding point anywhere (oracle/dit_fp32.py,
  ``pure=True``, TF32 off), evaluated on the GPU in fp32 for speed.

Measured per case and asserted against the tolerances stated here and in DESIGN.md §5.1:
every completion's latent (rel-RMS and max-abs relative to the oracle latent's RMS); the
per-step velocity magnitude ratio ||v_gpu|| / ||v_fp32|| at each of the 8 sigmas (both
evaluated at the GPU trajectory's inputs, so it isolates one forward's bf16 attenuation --
the effect PAPER.md:226 reports as ~7x under fp16 compounding, including t < 0.5); and the
ToyCodec (C=64, hop 1920) int16 audio of every completion, in LSB.  Cases: plain SDE,
full-cfg, onetime-negative, self-negative + APG, and 2-condition blended requests (the
unconditional and per-condition DiT rows).  A JSON summary of every metric is written to
gpurun_out/dit_trajectory.json when that directory exists.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

T, D, DEPTH, S = 1500, 64, 4, 8
TICKS = 18            # completions at ticks 7, 9, ...: 5 generations, the request changes at tick 6
SWITCH = 6

# Tolerances (bf16 operands, fp32 accumulation, 24 layers).  Measured on B200:
# latent rel-RMS 3.4e-3 .. 6.5e-3, max-abs 1.5-3.0% of the latent RMS; velocity norm ratio
# within 1 +- 2.1e-4 at every sigma (t = 1 .. 0.3), one-forward rel-RMS <= 5.6e-3; audio
# 22-53 LSB RMS (0.4-0.9% of the signal), max 307 LSB.  Bounds are ~2x the worst case
# (10x for the norm ratio, whose bound is the paper's attenuation concern).
TOL_LATENT_REL_RMS = 1.5e-2
TOL_LATENT_MAX_REL = 0.06       # max |diff| / rms(oracle latent)
TOL_VEL_RATIO = 2e-3            # | ||v_gpu|| / ||v_fp32|| - 1 | at every sigma
TOL_VEL_REL_RMS = 1.2e-2        # rms(v_gpu - v_fp32) / rms(v_fp32) per forward
TOL_AUDIO_RMS_LSB = 120.0       # rms of the int16 difference (full scale 32767)
TOL_AUDIO_REL = 2e-2            # rms(diff) / rms(oracle audio)

RESULTS: dict = {}


def _dump():
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "dit_trajectory.json"), "w") as fh:
            json.dump(RESULTS, fh, indent=1, sort_keys=True)


@pytest.fixture(scope="module")
def dm():
    from paper_2605_28657_b200 import dit

    return dit


@pytest.fixture(scope="module")
def dit8(dm):
    return dm.DiT(dm.DiTConfig(), frames=T, max_rows=2 * DEPTH)


@pytest.fixture(scope="module")
def codec():
    import oracle.ringflow_np as O

    return O.Codec(channels=D, hop=1920)


def _recording(dm):
    class Recording(dm.DiTVelocity):
        """DiTVelocity that keeps (inputs, timesteps, tokens, velocities) of every forward."""

        def __init__(self, dit):
            super().__init__(dit)
            self.log = []

        def forward(self, pipe):
            p = self._p
            xs, ts, conds = [x.clone() for x in p.xs], list(p.ts), list(p.conds)
            super().forward(pipe)
            if xs:
                self.log.append((xs, ts, conds, self.dit.out[:len(xs)].clone()))

    return Recording


def _requests(kind, text="bench prompt"):
    """(GPU request, oracle request) of one case, same content."""
    import scenarios

    import oracle.ringflow_np as O
    import paper_2605_28657_b200 as rf

    src = scenarios.keyed(0, "bench-source", (T, D))
    p1 = rf.content_hash("bench", text)
    if kind == "multi":
        p2 = rf.prompt_id("second prompt")
        w1, w2 = np.linspace(1.0, 0.2, T), np.linspace(0.1, 1.0, T)
        g = rf.GenerationRequest(conditions=(rf.ConditionSet(p1, source=src, weight_curve=w1),
                                             rf.ConditionSet(p2, hint_strength=0.5, weight_curve=w2)))
        o = O.Request([O.Cond(p1, source=src, weight=w1), O.Cond(p2, hint=0.5, weight=w2)])
        return g, o
    if kind == "sde":
        return (rf.GenerationRequest(conditions=(rf.ConditionSet(p1, source=src),)),
                O.Request([O.Cond(p1, source=src)]))
    mode, scale, apg = {"full-cfg": ("full-cfg", 3.0, None), "onetime": ("onetime-negative", 2.5, None),
                        "selfneg-apg": ("self-negative", 2.0, 0.5)}[kind]
    curves = {"guidance_curve": np.full(T, scale)}
    if apg is not None:
        curves["apg_momentum"] = np.full(T, apg)
    g = rf.GenerationRequest(conditions=(rf.ConditionSet(p1, source=src),),
                             curves=rf.make_curves(T, guidance_enabled=True, rcfg_mode=mode, **curves))
    o = O.Request([O.Cond(p1, source=src)], curves=curves, guidance=True, rcfg=mode)
    return g, o


def _rel_rms(a, b):
    return float(np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2)))


def _run_case(dm, dit, codec, kind):
    import oracle.ringflow_np as O
    import paper_2605_28657_b200 as rf
    from oracle.dit_fp32 import Fp32DiTVelocity, reference_forward

    greq, oreq = _requests(kind)
    vel = _recording(dm)(dit)
    pipe = rf.StreamPipeline(rf.PipelineConfig(depth=DEPTH, steps=S, frames=T, channels=D, seed=0), request=greq,
                             velocity_model=vel)
    ref = O.Pipeline(depth=DEPTH, steps=S, frames=T, channels=D, seed=0, request=oreq)
    ref.model = Fp32DiTVelocity(dit)
    recs, orecs = [], []
    g2, o2 = _requests(kind, "bench prompt, second")
    for k in range(TICKS):
        if k == SWITCH:   # later generations differ from the first ones
            pipe.set_request(g2)
            ref.set_request(o2)
        recs += pipe.tick()
        orecs += ref.tick()
        assert pipe.last_timesteps == ref.last_timesteps   # bit-exact per-row timestep gather
    torch.cuda.synchronize()
    assert len(recs) == len(orecs) >= 5
    out = {"completions": len(recs), "latent": [], "audio": [], "velocity_by_sigma": {}}
    for r, o in zip(recs, orecs):
        assert (r.tick, r.completion_index, r.submission_id, r.schedule_id) == \
            (o.tick, o.completion_index, o.submission_id, o.schedule_id)
        a, b = r.latent, o.latent
        assert np.isfinite(a).all()
        scale = float(np.sqrt(np.mean(b ** 2)))
        out["latent"].append({"rel_rms": _rel_rms(a, b), "max_abs_over_rms": float(np.max(np.abs(a - b)) / scale),
                              "oracle_rms": scale})
        pa, pb = codec.full(a).astype(np.float64), codec.full(b).astype(np.float64)
        d = pa - pb
        out["audio"].append({"rms_lsb": float(np.sqrt(np.mean(d ** 2))), "max_lsb": float(np.max(np.abs(d))),
                             "rel_rms": float(np.sqrt(np.mean(d ** 2)) / max(np.sqrt(np.mean(pb ** 2)), 1.0)),
                             "frac_samples_differ": float(np.mean(d != 0)),
                             "oracle_rms_lsb": float(np.sqrt(np.mean(pb ** 2)))})
    # one-forward attenuation at each sigma: the fp32 network at the GPU trajectory's inputs
    by_t: dict = {}
    for xs, ts, conds, v in vel.log:
        ref_v = reference_forward(dit, xs, ts, conds, pure=True)
        for i, t in enumerate(ts):
            vg, vr = v[i].double(), ref_v[i].double()
            ratio = float(vg.norm() / vr.norm())
            err = float((vg - vr).pow(2).mean().sqrt() / vr.pow(2).mean().sqrt())
            by_t.setdefault(round(float(t), 6), []).append((ratio, err))
    for t, vals in sorted(by_t.items()):
        out["velocity_by_sigma"][str(t)] = {"ratio_min": min(v[0] for v in vals), "ratio_max": max(v[0] for v in vals),
                                            "rel_rms_max": max(v[1] for v in vals), "forwards": len(vals)}
    RESULTS[kind] = out
    _dump()
    return out


@pytest.mark.parametrize("kind", ["sde", "full-cfg", "onetime", "selfneg-apg", "multi"])
def test_trajectory_vs_pure_fp32(dm, dit8, codec, kind):
    out = _run_case(dm, dit8, codec, kind)
    sig = sorted(float(t) for t in out["velocity_by_sigma"])
    assert len(sig) == S and min(sig) < 0.5          # all eight sigmas seen, incl. t < 0.5
    for t, v in out["velocity_by_sigma"].items():
        assert abs(v["ratio_min"] - 1.0) <= TOL_VEL_RATIO and abs(v["ratio_max"] - 1.0) <= TOL_VEL_RATIO, (t, v)
        assert v["rel_rms_max"] <= TOL_VEL_REL_RMS, (t, v)
    for lat in out["latent"]:
        assert lat["rel_rms"] <= TOL_LATENT_REL_RMS, lat
        assert lat["max_abs_over_rms"] <= TOL_LATENT_MAX_REL, lat
    for au in out["audio"]:
        assert au["rms_lsb"] <= TOL_AUDIO_RMS_LSB and au["rel_rms"] <= TOL_AUDIO_REL, au


def test_model_weights_swap_on_dit_path(dm, codec):
    """set_model_weights under DiTVelocity: the shared style offset enters every DiT
    velocity in x0 space (v - style / t, reference model.py:123-131 + pipeline.py:332-337),
    visible from the next tick (acceptance C06: effect at the first post-write completion),
    and the GPU trajectory stays within the fp32 tolerance of the oracle doing the same."""
    import scenarios

    import oracle.ringflow_np as O
    import paper_2605_28657_b200 as rf
    from oracle.dit_fp32 import Fp32DiTVelocity

    cfg = dm.DiTConfig().small()
    Ts = 96
    dit = dm.DiT(cfg, frames=Ts, max_rows=4)
    src = scenarios.keyed(3, "src", (Ts, D))
    p1 = rf.prompt_id("weights")
    pipe = rf.StreamPipeline(rf.PipelineConfig(depth=4, steps=S, frames=Ts, channels=D),
                             request=rf.GenerationRequest(conditions=(rf.ConditionSet(p1, source=src),)),
                             velocity_model=dm.DiTVelocity(dit))
    ref = O.Pipeline(depth=4, steps=S, frames=Ts, channels=D, request=O.Request([O.Cond(p1, source=src)]))
    ref.model = Fp32DiTVelocity(dit)
    offset = 0.5 * scenarios.keyed(9, "offset", (Ts, D))
    recs, orecs = [], []
    for k in range(30):
        if k == 16:
            assert pipe.set_model_weights(offset) == pipe.tick_index
            ref.set_model_weights(offset)
        recs += pipe.tick()
        orecs += ref.tick()
    assert len(recs) == len(orecs)
    post = [i for i, r in enumerate(recs) if r.tick >= 16]
    assert recs[post[0]].rms_vs_reference > 0.0              # effect at post-write completion 0
    assert all(recs[i].rms_vs_reference is None for i in range(post[0]) if recs[i].tick < 16)
    for r, o in zip(recs, orecs):
        assert _rel_rms(r.latent, o.latent) <= TOL_LATENT_REL_RMS
        if o.rms_vs_reference is not None:
            assert abs(r.rms_vs_reference - o.rms_vs_reference) <= 0.05 * o.rms_vs_reference + 1e-9


def test_config5_dit_forward_vs_fp32(dm):
    """240-s latent (config 5: T=6000 -> 3000 tokens): one batched forward of 4 rows at
    distinct timesteps (incl. t < 0.5) against the bf16-rounding oracle (same rounding
    points: accumulation-order differences only) and the pure fp32 network."""
    from oracle.dit_fp32 import reference_forward

    frames = 6000
    dit = dm.DiT(dm.DiTConfig(), frames=frames, max_rows=4)
    g = torch.Generator(device="cuda").manual_seed(60)
    xs = [torch.randn(frames, D, device="cuda", generator=g, dtype=torch.float64) for _ in range(4)]
    ts = [1.0, 0.75, 0.5, 0.3]
    conds = [dit.cond_tokens(2000 + i) for i in range(4)]
    out = dit.forward(xs, ts, conds).clone()
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    rounded = reference_forward(dit, xs, ts, conds)
    pure = reference_forward(dit, xs, ts, conds, pure=True)
    res = {"rel_rms_vs_bf16_rounding_oracle": [], "rel_rms_vs_pure_fp32": [], "norm_ratio_vs_pure_fp32": []}
    for i in range(4):
        a, b, c = out[i].double(), rounded[i].double(), pure[i].double()
        res["rel_rms_vs_bf16_rounding_oracle"].append(float((a - b).pow(2).mean().sqrt() / b.pow(2).mean().sqrt()))
        res["rel_rms_vs_pure_fp32"].append(float((a - c).pow(2).mean().sqrt() / c.pow(2).mean().sqrt()))
        res["norm_ratio_vs_pure_fp32"].append(float(a.norm() / c.norm()))
    RESULTS["config5_forward"] = res
    _dump()
    assert max(res["rel_rms_vs_bf16_rounding_oracle"]) < 1e-2
    assert max(res["rel_rms_vs_pure_fp32"]) < TOL_VEL_REL_RMS
    assert all(abs(r - 1.0) <= TOL_VEL_RATIO for r in res["norm_ratio_vs_pure_fp32"])
