"""Scripted pipeline scenarios, runnable against any implementation of the ringflow API.

``drive(api, spec)`` runs one scenario through a module exposing the reference's public
names (the real reference ``ringflow`` when generating goldens in the build container,
or ``paper_2605_28657_b200`` on the GPU) and returns a flat dict of numpy arrays.
``drive_oracle(spec)`` does the same through the CPU oracle (oracle/ringflow_np.py).
Inputs (sources, targets, offsets, curves) are generated from keyed numpy Philox draws
here, identically for every implementation.
"""
from __future__ import annotations

import numpy as np


def keyed(seed, tag, shape):
    """Input fixture: the reference's own NoiseSource(seed).normal(0, tag, shape) recipe."""
    import hashlib
    import struct

    h = hashlib.blake2b(digest_size=16)
    h.update(struct.pack("<qq", seed, 0))
    h.update((0).to_bytes(16, "little", signed=True))
    h.update(tag.encode("utf-8"))
    key = int.from_bytes(h.digest(), "little")
    return np.random.Generator(np.random.Philox(key=key)).standard_normal(shape)


def _sweep(n):
    down = [1.0 - 0.5 * i / 30 for i in range(31)]
    up = [0.5 + 0.5 * j / 29 for j in range(1, 30)]
    return (down + up)[:n]


# Each spec: config kwargs, request recipe, and a list of ops.
SPECS = {
    # BASELINE config 1: T=250 (10 s at 25 Hz), D=8, depth 4, S=4
    "c1_default": dict(config=dict(depth=4, steps=4, frames=250, channels=8), request=dict(prompt="c1", source="src"),
                       ops=[("tick", 24)]),
    "c1_denoise": dict(config=dict(depth=4, steps=4, frames=250, channels=8, denoise=0.6),
                       request=dict(prompt="c1", source="src"), ops=[("tick", 12), ("set_denoise", 0.9), ("tick", 12)]),
    "shared_sde_curve": dict(config=dict(depth=8, steps=8), request=dict(prompt="p", source="src", sde=0.1),
                             ops=[("tick", 24), ("set_shared_curve", "sde_denoise_curve", 0.95), ("tick", 17)]),
    "migration": dict(config=dict(depth=8, steps=8, mode="migration"), request=dict(prompt="p", source="src"),
                      ops=[("tick", 24), ("set_denoise", 0.5), ("tick", 12)]),
    "global_reset_sweep": dict(config=dict(depth=8, steps=8, mode="global-reset"), request=dict(prompt="p", source="src"),
                               ops=[("tick", 24), ("sweep", 20), ("tick", 8)]),
    "per_slot_sweep": dict(config=dict(depth=4, steps=8), request=dict(prompt="p", source="src"),
                           ops=[("tick", 16), ("sweep", 24)]),
    "per_frame_blend": dict(config=dict(depth=4, steps=8, denoise=0.7), request=dict(prompt="p", source="src", sde="ramp"),
                            ops=[("tick", 8), ("modulate", 16)]),
    "x0_morph": dict(config=dict(depth=8, steps=8), request=dict(prompt="p", source="src", hint=1.0),
                     ops=[("tick", 24), ("set_shared_curve", "x0_target", "target"), ("tick", 10),
                          ("set_shared_curve", "x0_target_strength", "ramp"), ("tick", 10)]),
    "weight_swap": dict(config=dict(depth=2, steps=8), request=dict(prompt="p", timbre=1.0),
                        ops=[("tick", 20), ("set_model_weights", "offset"), ("tick", 12)]),
    "ode_curves": dict(config=dict(depth=4, steps=8), request=dict(prompt="p", solver="ode", vscale="ramp", ode_noise=0.2,
                                                                   x0_target="target"),
                       ops=[("tick", 20)]),
    "guidance_full": dict(config=dict(depth=4, steps=8), request=dict(prompt="p", source="src", guidance="full-cfg",
                                                                      gscale=3.0),
                          ops=[("tick", 20)]),
    "guidance_onetime": dict(config=dict(depth=4, steps=8), request=dict(prompt="p", source="src",
                                                                         guidance="onetime-negative", gscale=2.0),
                             ops=[("tick", 20)]),
    "guidance_self_apg": dict(config=dict(depth=4, steps=8), request=dict(prompt="p", source="src", guidance="self-negative",
                                                                          gscale=2.5, apg=0.5),
                              ops=[("tick", 20)]),
    "guidance_rescale": dict(config=dict(depth=4, steps=8), request=dict(prompt="p", source="src", guidance="off",
                                                                         gscale=4.0, rescale=0.7),
                             ops=[("tick", 20)]),
    "multi_cond": dict(config=dict(depth=4, steps=8), request=dict(prompt="p", source="src", multi=True),
                       ops=[("tick", 20)]),
    "no_jitter": dict(config=dict(depth=4, steps=4, model_jitter=0.0), request=dict(prompt="p", source="src"),
                      ops=[("tick", 12)]),
    "wide_channels": dict(config=dict(depth=4, steps=8, frames=40, channels=64), request=dict(prompt="w", source="src"),
                          ops=[("tick", 20)]),
    "mode_switch": dict(config=dict(depth=8, steps=8), request=dict(prompt="p", source="src"),
                        ops=[("tick", 24), ("set_mode", "migration"), ("set_denoise", 0.8), ("tick", 4),
                             ("set_mode", "per-slot"), ("tick", 12)]),
}


def _inputs(spec):
    cfg = dict(dict(frames=96, channels=8), **spec["config"])
    T, D = cfg["frames"], cfg["channels"]
    return T, D, {
        "src": keyed(100, "source", (T, D)),
        "src2": keyed(101, "source2", (T, D)),
        "target": keyed(55, "target", (T, D)),
        "offset": 0.5 * keyed(77, "offset", (T, D)),
        "ramp": np.linspace(0.0, 1.0, T),
        "wramp": np.linspace(0.2, 1.0, T),
    }


def _curve_arg(val, inputs):
    return inputs[val] if isinstance(val, str) else val


def _build_request(api, spec, inputs, T):
    r = spec["request"]
    src = inputs[r["source"]] if r.get("source") else None
    ph = api.prompt_id(r["prompt"])
    conds = [api.ConditionSet(prompt_hash=ph, hint_strength=r.get("hint", 0.0),
                              timbre_strength=r.get("timbre", 0.0), source=src,
                              weight_curve=inputs["wramp"] if r.get("multi") else None)]
    if r.get("multi"):
        conds.append(api.ConditionSet(prompt_hash=api.prompt_id("second"), hint_strength=0.5,
                                      weight_curve=1.0 - inputs["ramp"] * 0.5))
    named = {}
    if "sde" in r:
        named["sde_denoise_curve"] = _curve_arg(r["sde"], inputs)
    if "vscale" in r:
        named["velocity_scale"] = _curve_arg(r["vscale"], inputs) + 0.5
    if "ode_noise" in r:
        named["ode_noise_curve"] = r["ode_noise"]
    if "gscale" in r:
        named["guidance_curve"] = r["gscale"]
    if "apg" in r:
        named["apg_momentum"] = r["apg"]
    if "rescale" in r:
        named["cfg_rescale_curve"] = r["rescale"]
    curves = api.make_curves(T, x0_target=inputs[r["x0_target"]] if r.get("x0_target") else None,
                             guidance_enabled="guidance" in r, rcfg_mode=r.get("guidance", "off"), **named)
    return api.GenerationRequest(conditions=tuple(conds), curves=curves, solver=r.get("solver", "sde"))


def _modulated(T, k):
    return np.clip(np.linspace(0.0, 1.0, T) * (0.5 + 0.5 * np.sin(2 * np.pi * k / 16)), 0.0, 1.0)


def drive(api, spec):
    """Run a scenario through a ringflow-API module; returns flat trace arrays."""
    T, D, inputs = _inputs(spec)
    cfg = api.PipelineConfig(**dict(dict(frames=96, channels=8), **spec["config"]))
    kw = {"noise_cache_bytes": spec["noise_cache_bytes"]} if "noise_cache_bytes" in spec else {}
    pipe = api.StreamPipeline(cfg, request=_build_request(api, spec, inputs, T), **kw)
    recs, ticks_ts, snaps = [], [], []

    def run(n):
        for _ in range(n):
            for rec in pipe.tick():
                recs.append(rec)
            ticks_ts.append([(float(s), i) for s, i in pipe.last_timesteps])
            snaps.append(snapshot_str(pipe.snapshot()))

    for op in spec["ops"]:
        kind = op[0]
        if kind == "tick":
            run(op[1])
        elif kind == "set_denoise":
            pipe.set_denoise(op[1])
        elif kind == "set_mode":
            pipe.set_mode(op[1])
        elif kind == "set_shared_curve":
            pipe.set_shared_curve(op[1], _curve_arg(op[2], inputs))
        elif kind == "set_model_weights":
            pipe.set_model_weights(inputs[op[1]])
        elif kind == "sweep":
            for v in _sweep(op[1]):
                pipe.set_denoise(v)
                run(1)
        elif kind == "modulate":
            for k in range(op[1]):
                pipe.set_shared_curve("sde_denoise_curve", _modulated(T, k))
                run(1)
        else:
            raise ValueError(kind)
    return _trace(recs, ticks_ts, pipe, snaps)


def snapshot_str(snap) -> str:
    """Canonical text of a PipelineSnapshot (reference pipeline.py:221-244, 289-304): every
    field, floats by repr, so equal strings mean equal snapshots."""
    slots = ";".join("-" if v is None else f"{float(v.denoise)!r},{int(v.step)},{v.schedule_id}" for v in snap.slots)
    vals = ",".join(repr(float(d)) for d in sorted(snap.denoise_values()))
    return f"{snap.tick}|{snap.mode}|{float(snap.denoise)!r}|{snap.queue_depth}|{slots}|{vals}"


def _trace(recs, ticks_ts, pipe, snaps):
    n = len(recs)
    out = {
        "snapshot": np.array(snaps, dtype=object).astype(str),
        "tick": np.array([r.tick for r in recs], dtype=np.int64),
        "completion_index": np.array([r.completion_index for r in recs], dtype=np.int64),
        "submission_id": np.array([r.submission_id for r in recs], dtype=np.int64),
        "schedule_id": np.array([r.schedule_id for r in recs], dtype="U12"),
        "denoise": np.array([r.denoise for r in recs], dtype=np.float64),
        "hybrid": np.array([r.hybrid for r in recs], dtype=bool),
        "decode_skipped": np.array([r.decode_skipped for r in recs], dtype=bool),
        "rms": np.array([np.nan if r.rms_vs_reference is None else r.rms_vs_reference for r in recs]),
        "latents": np.stack([np.asarray(r.latent) for r in recs]) if n else np.zeros((0,)),
        "ts_count": np.array([len(t) for t in ticks_ts], dtype=np.int64),
        "ts_sigma": np.array([s for t in ticks_ts for s, _ in t], dtype=np.float64),
        "ts_id": np.array([i for t in ticks_ts for _, i in t], dtype="U12"),
        "final_tick": np.array(pipe.tick_index),
        "completions_total": np.array(pipe.completions_total),
    }
    return out


def drive_oracle(spec):
    """Same scenario through the CPU oracle restatement."""
    import oracle.ringflow_np as O

    T, D, inputs = _inputs(spec)
    c = dict(dict(frames=96, channels=8), **spec["config"])
    r = spec["request"]
    src = inputs[r["source"]] if r.get("source") else None
    conds = [O.Cond(O.prompt_id(r["prompt"]), r.get("hint", 0.0), r.get("timbre", 0.0), src,
                    inputs["wramp"] if r.get("multi") else None)]
    if r.get("multi"):
        conds.append(O.Cond(O.prompt_id("second"), 0.5, 0.0, None, 1.0 - inputs["ramp"] * 0.5))
    curves = {}
    if "sde" in r:
        curves["sde_denoise_curve"] = O.clamp("sde_denoise_curve", _curve_arg(r["sde"], inputs), T)
    if "vscale" in r:
        curves["velocity_scale"] = O.clamp("velocity_scale", _curve_arg(r["vscale"], inputs) + 0.5, T)
    if "ode_noise" in r:
        curves["ode_noise_curve"] = O.clamp("ode_noise_curve", r["ode_noise"], T)
    if "gscale" in r:
        curves["guidance_curve"] = O.clamp("guidance_curve", r["gscale"], T)
    if "apg" in r:
        curves["apg_momentum"] = O.clamp("apg_momentum", r["apg"], T)
    if "rescale" in r:
        curves["cfg_rescale_curve"] = O.clamp("cfg_rescale_curve", r["rescale"], T)
    req = O.Request(conds, curves, r.get("solver", "sde"), inputs[r["x0_target"]] if r.get("x0_target") else None,
                    "guidance" in r, r.get("guidance", "off"))
    pipe = O.Pipeline(depth=c["depth"], steps=c["steps"], frames=c["frames"], channels=c["channels"],
                      mode=c.get("mode", "per-slot"), seed=c.get("seed", 0), denoise=c.get("denoise", 1.0),
                      jitter=c.get("model_jitter", 0.1), request=req)
    recs, ticks_ts, snaps = [], [], []

    def run(n):
        for _ in range(n):
            recs.extend(pipe.tick())
            ticks_ts.append([(float(s), i) for s, i in pipe.last_timesteps])
            snaps.append(snapshot_str(pipe.snapshot()))

    for op in spec["ops"]:
        kind = op[0]
        if kind == "tick":
            run(op[1])
        elif kind == "set_denoise":
            pipe.set_denoise(op[1])
        elif kind == "set_mode":
            pipe.set_mode(op[1])
        elif kind == "set_shared_curve":
            pipe.set_shared_curve(op[1], _curve_arg(op[2], inputs))
        elif kind == "set_model_weights":
            pipe.set_model_weights(inputs[op[1]])
        elif kind == "sweep":
            for v in _sweep(op[1]):
                pipe.set_denoise(v)
                run(1)
        elif kind == "modulate":
            for k in range(op[1]):
                pipe.set_shared_curve("sde_denoise_curve", _modulated(T, k))
                run(1)

    class _P:
        tick_index = pipe.tick_index
        completions_total = pipe.completions

    return _trace(recs, ticks_ts, _P, snaps)


# fields compared bit-exactly (integer / id / flag bookkeeping)
EXACT_FIELDS = ("tick", "completion_index", "submission_id", "schedule_id", "denoise", "hybrid",
                "decode_skipped", "ts_count", "ts_sigma", "ts_id", "final_tick", "completions_total", "snapshot")
