"""CPU-only checks: the C ABI library loads and exports its header; host bookkeeping."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

import oracle.ringflow_np as O
import paper_2605_28657_b200 as rf
from paper_2605_28657_b200 import _native, build
from paper_2605_28657_b200.latents import philox_key

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            names |= set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(rf_\w+)\s*\(", src, re.M))
    return names


def test_library_builds_and_exports_header():
    path = build.build()
    lib = ctypes.CDLL(path)
    declared = header_functions()
    assert declared >= {"rf_normal_fill", "rf_tick_solve", "rf_emit_stats", "rf_decode_window"}
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_native.EXPORTS) == declared
    lib.rf_abi_version.restype = ctypes.c_int
    assert lib.rf_abi_version() == 1


def test_sm100a_code_in_library():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2605_28657_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(^|\n)\s*(from|import)\s+oracle\b|liboracle|oracle/_build|"
                                     r"ringflow_np|oracle/npyrandom", src), f


def test_device_required_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2605_28657_b200._device import NoDeviceError

    with pytest.raises(NoDeviceError):
        rf.NoiseSource(0).normal(0, "x", (4,))


def test_schedule_matches_oracle():
    for d in (1.0, 0.5, 0.3, 1e-4):
        for s in (1, 3, 8, 16):
            sc = rf.build_schedule(d, s, 3.0)
            assert np.array_equal(sc.sigmas, O.sigmas_of(d, s, 3.0))
            assert sc.schedule_id == O.schedule_id(O.sigmas_of(d, s, 3.0), 3.0)
    c = rf.ScheduleCache()
    assert c.get(0.5, 8, 3.0) is c.get(0.5 + 1e-8, 8, 3.0)
    with pytest.raises(rf.ScheduleMismatchError):
        rf.migrate_schedule(rf.build_schedule(1.0, 8), 3, rf.build_schedule(1.0, 4))
    with pytest.raises(ValueError):
        rf.build_schedule(0.0, 8)


def test_hashes_match_oracle():
    parts = ("prompt", 3, 2.5, None, True, b"xy", [1, (2, "z")], np.arange(6.0).reshape(2, 3))
    assert rf.content_hash(*parts) == O.chash(*parts)
    assert rf.content_hash(torch.arange(6.0, dtype=torch.float64).reshape(2, 3)) == \
        O.chash(np.arange(6.0).reshape(2, 3))
    assert rf.prompt_id("steady prompt") == O.prompt_id("steady prompt")
    for args in [(0, 0, 0, "sde"), (2**40, -5, 7, "model"), (1, 2**62, 3, "init")]:
        assert philox_key(*args) == O.philox_key(*args)
    with pytest.raises(ValueError):
        philox_key(0, 0, -1, "x")


def test_curve_plumbing():
    assert rf.clamp_curve("guidance_curve", 12.0, 5).tolist() == [8.0] * 5
    with pytest.raises(KeyError):
        rf.clamp_curve("nope", 1.0, 4)
    with pytest.raises(rf.ShapeMismatchError):
        rf.clamp_curve("velocity_scale", np.ones(5), 4)
    bad = np.ones(4)
    bad[1] = np.inf
    with pytest.raises(ValueError):
        rf.clamp_curve("velocity_scale", bad, 4)
    with pytest.raises(ValueError):
        rf.make_curves(4, x0_target_strength=1.0)
    assert rf.sentinel("apg_momentum", 3).tolist() == [0, 0, 0]
    assert rf.sentinel("cfg_rescale_curve", 2).tolist() == [1, 1]


def test_config_and_request_validation():
    with pytest.raises(ValueError):
        rf.PipelineConfig(depth=0)
    with pytest.raises(ValueError):
        rf.PipelineConfig(mode="nope")
    with pytest.raises(ValueError):
        rf.PipelineConfig(denoise=1.5)
    with pytest.raises(ValueError):
        rf.GenerationRequest(conditions=())
    with pytest.raises(ValueError):
        rf.GenerationRequest(conditions=(rf.ConditionSet(1),), solver="euler")
    with pytest.raises(ValueError):
        rf.ConditionSet(1, hint_strength=2.0)
    a = rf.ConditionSet(5, 0.5, 0.0, np.ones((3, 2)))
    b = O.Cond(5, 0.5, 0.0, np.ones((3, 2)))
    assert a.content_key() == b.content_key()
    r = rf.GenerationRequest(conditions=(a,), solver="ode")
    assert r.content_key() == O.Request([b], solver="ode").content_key()


def test_bench_reference_arm_json_contract():
    """`bench.py --impl reference` (the CPU arm the driver runs): one JSON line on the same
    metric / unit as our arm, impl "reference", a cpu_baseline describing the run and an e2e
    object with zero host<->device bytes; the sample is the config-2 workload (DiT in the
    reference tick's model slot) and the reference's toy model is reported beside it."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    import bench

    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["higher_is_better"] is True and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["ticks"] >= 1 and "DiT" in line["cpu_baseline"]["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": bench.UNIT, "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["toy_model"]["value"] > 0
