#!/usr/bin/env python
"""Benchmark: decoder completions/s for 60-s music at ring depth 4, S=8 (BASELINE config 2).

A step is one ``StreamPipeline.tick()`` of the ring (T=1500 latent frames at 25 Hz,
D=64 channels, depth 4, S=8, source present, denoise 1.0); at depth 4 / S=8 the ring
completes one generation every 2 ticks.  value = completions of all ranks / max-over-
ranks device time (CUDA events on the pipeline's stream around each tick; L2 flushed
between ticks outside the timed events).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun: each rank drives its own independent stream (its own ring,
seed = rank): weak scaling, no data-path collective.  --impl reference times the
reference's CPU path (the oracle port oracle/ringflow_np.py, float64 numpy) on the
host cores, one independent stream per process.
"""
from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "decoder completions/sec, 60-s music, depth 4 S=8; windowed decode ms; %roofline"
UNIT = "completions/s"
T, D, DEPTH, STEPS = 1500, 64, 4, 8
HOP, WINDOW, OVERLAP = 1920, 75, 15   # 48 kHz, 3-s playback window (service.py:315-322), RF=15
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=32)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ------------------------------------------------------------------- clocks -----
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            # one synchronous sample at the end so a short timed region still has data
            try:
                snap = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                      timeout=20).stdout
            except Exception:
                snap = ""
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()
            with open(self.path, "a") as fh:
                fh.write(snap)

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workload -----
def make_request(rf, stream_id):
    import scenarios

    src = scenarios.keyed(stream_id, "bench-source", (T, D))
    cond = rf.ConditionSet(prompt_hash=rf.content_hash("bench", "bench prompt"), source=src)
    return rf.GenerationRequest(conditions=(cond,))


def solve_bytes_per_row():
    # rf_tick_kernel touches, per element (float64): x read+write, x0 partial, style
    # offset, model noise, sde noise, source = 7 x 8 B (no curves at config 2).
    return T * D * 7 * 8


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_28657_b200 as rf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    pipe = rf.StreamPipeline(rf.PipelineConfig(depth=DEPTH, steps=STEPS, frames=T, channels=D, seed=rank),
                             request=make_request(rf, rank))
    st = pipe.stream
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def flush_l2():
        with torch.cuda.stream(st):
            flush.fill_(1)

    for _ in range(args.warmup):
        pipe.tick()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- device-timed run (kernel-resident inputs) ----
    pairs, completions, launches = [], 0, 0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush_l2()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            recs = pipe.tick()
            b.record(st)
            pairs.append((a, b))
            completions += len(recs)
            launches += pipe.launches_last_tick
        torch.cuda.synchronize()
    dev_ms = sum(a.elapsed_time(b) for a, b in pairs)
    clocks = clk.summary()

    # ---- roofline of the dominant kernel (fused solve) ----
    phases = pipe.enable_phase_timing(True)
    for _ in range(args.steps):
        flush_l2()
        pipe.tick()
    torch.cuda.synchronize()
    pipe.enable_phase_timing(False)
    phase_ms = {k: sum(a.elapsed_time(b) for a, b in v) / len(v) for k, v in phases.items()}
    rows = DEPTH  # steady state: every slot active each tick
    solve_bytes = rows * solve_bytes_per_row()
    hbm_peak, _, peak_src = peaks()
    achieved = solve_bytes / (phase_ms["solve"] * 1e-3) / 1e9

    # ---- end-to-end through the public API with host buffers ----
    curve_host = torch.from_numpy(np.clip(np.linspace(0.0, 1.0, T), 0, 1)).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_done, h2d, d2h = 0, 0, 0
    for k in range(args.steps):
        # per-tick control input from pinned host memory (config 4-style shared write)
        pipe.set_shared_curve("sde_denoise_curve", 1.0 if k % 2 else 0.999)
        h2d += T * 8
        for r in pipe.tick():
            _ = r.latent   # device -> host copy of the completion
            d2h += T * D * 8
            e2e_done += 1
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    del curve_host

    # ---- windowed decode (3-s window + overlap 15) of the last completion ----
    codec = rf.ToyCodec(channels=D, hop=HOP)
    lat = pipe._last_emitted  # device float64 [T, D]
    with torch.cuda.stream(st):
        for _ in range(5):
            codec.decode_device(lat, T - WINDOW, T, OVERLAP, False)
        ev = []
        for _ in range(20):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            codec.decode_device(lat, T - WINDOW, T, OVERLAP, False)
            b.record(st)
            ev.append((a, b))
    torch.cuda.synchronize()
    decode_ms = sum(a.elapsed_time(b) for a, b in ev) / len(ev)

    # ---- aggregate over ranks ----
    tot = torch.tensor([completions, dev_ms, e2e_done, e2e_s, launches], dtype=torch.float64, device=dev)
    if world > 1:
        s = tot.clone()
        m = tot.clone()
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        completions_all, dev_ms_max, e2e_all, e2e_max = s[0].item(), m[1].item(), s[2].item(), m[3].item()
    else:
        completions_all, dev_ms_max, e2e_all, e2e_max = completions, dev_ms, e2e_done, e2e_s
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    value = completions_all / (dev_ms_max * 1e-3)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dev_ms_max / args.steps, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config 2: 60-s latent T=1500 x D=64, ring depth 4, S=8, toy velocity model, "
                               "source present, denoise 1.0; one independent stream per GPU",
                   "frames": T, "channels": D, "depth": DEPTH, "steps_per_generation": STEPS,
                   "l2": "flushed (256 MiB write) between timed ticks, outside the events",
                   "completions_timed": int(completions_all)},
        "e2e": {"value": round(e2e_all / e2e_max, 3), "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps,
                "note": "wall clock through StreamPipeline: per-tick shared-curve write from host, "
                        "CompletionRecord.latent read back to host"},
        "windowed_decode_ms": round(decode_ms, 5),
        "phase_ms": {k: round(v, 5) for k, v in phase_ms.items()},
        "roofline": {"bound": "hbm", "kernel": "rf_tick_kernel", "achieved": round(achieved, 1), "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": None,
                     "algorithmic_bytes_per_launch": solve_bytes, "peak_source": peak_src},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds, processes=1)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------- CPU reference arm -----
def _oracle_worker(args):
    stream_id, seconds, warm = args
    import scenarios

    import oracle.ringflow_np as O

    src = scenarios.keyed(stream_id, "bench-source", (T, D))
    req = O.Request([O.Cond(O.chash("bench", "bench prompt"), source=src)])
    pipe = O.Pipeline(depth=DEPTH, steps=STEPS, frames=T, channels=D, seed=stream_id, request=req)
    for _ in range(warm):
        pipe.tick()
    done, ticks = 0, 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        done += len(pipe.tick())
        ticks += 1
    return done, ticks, time.perf_counter() - t0


def cpu_baseline(seconds, processes=1):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if processes == 1:
        res = [_oracle_worker((0, seconds, 4 * STEPS))]
    else:
        with mp.get_context("spawn").Pool(processes) as pool:
            res = pool.map(_oracle_worker, [(i, seconds, 4 * STEPS) for i in range(processes)])
    done = sum(r[0] for r in res)
    ticks = sum(r[1] for r in res)
    wall = max(r[2] for r in res)
    return {"value": round(done / wall, 3), "unit": UNIT, "cores": processes, "kind": "port",
            "sample": f"oracle/ringflow_np.py StreamPipeline restatement, config 2 (T=1500, D=64, depth 4, S=8), "
                      f"{processes} independent stream(s), {ticks} warm ticks after {4 * STEPS} warmup, "
                      f"{wall:.1f} s wall, float64 numpy, 1 thread/process"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    per_step = max(1.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    base = cpu_baseline(per_step * args.steps, processes=procs)
    line = {
        "metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": "config 2: 60-s latent T=1500 x D=64, ring depth 4, S=8, toy velocity model "
                               "(the reference's only model), source present; one stream per host core"},
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
