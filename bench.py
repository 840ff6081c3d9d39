#!/usr/bin/env python
"""Benchmark: decoder completions/s for 60-s music at ring depth 4, S=8 (BASELINE config 2).

A step is one ``StreamPipeline.tick()`` of the ring: T=1500 latent frames (60 s at 25 Hz),
D=64 channels, depth 4, S=8, source present, denoise 1.0, SDE re-noise solver.  The
velocity model is the ACE-Step-1.5-shape 24-layer DiT (config 2; ``paper_2605_28657_b200.dit``,
random init, bf16 operands / fp32 accumulation); every tick runs ONE batched DiT forward
over the 4 ring rows, each at its own timestep, then the fused solver.  At depth 4 / S=8
the ring completes one generation every 2 ticks.

  value     = completions of all ranks / max-over-ranks device time (CUDA events on the
              pipeline stream around each tick; L2 flushed between ticks, outside events)
  e2e       = the same through the public API with host buffers: per-tick shared-curve
              write from host memory, every CompletionRecord.latent read back to host
  toy_path  = the same ring with the reference's own ToyFlowModel as velocity model (the
              only model the reference has); compare with cpu_baseline_toy_model
  cpu_baseline / --impl reference = the same config-2 workload on the host CPU: the
              reference's tick (oracle port, float64 numpy) with the DiT (oracle/dit_fp32.py,
              torch CPU, bf16 GEMM/attention operands, all host threads) in its model slot;
              the reference arm also reports the reference's toy model on all cores (`toy_model`)
  library_baseline = the same DiT forward in stock PyTorch (cuBLAS + SDPA) on the GPU

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: every rank drives its own independent stream (own ring and DiT, seed = rank):
weak scaling, no data-path collective; the only collective is config 5's sharded long
decode (NCCL all-gather of the PCM).  Launched under torchrun by the driver; started
plainly with --gpus N > 1 it re-executes itself under torch.distributed.run with N ranks.
`--stub` runs the same launch / aggregation / JSON path on the CPU over gloo with a stub
workload (harness test only: tests/test_bench_harness.py; never a bench number).
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import socket
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
    ap.add_argument("--steps", type=int, default=96)   # ~0.9 s of ticks: the power-capped steady state
    ap.add_argument("--warmup", type=int, default=24)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-toy", action="store_true")
    ap.add_argument("--no-library-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-240s-dit", action="store_true")
    ap.add_argument("--stub", action="store_true", help="CPU/gloo harness test with a stub workload")
    return ap.parse_args()


# ------------------------------------------------------------ launch / ranks -----
def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def maybe_respawn(args) -> None:
    """--gpus N > 1 without a torchrun environment: re-execute under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and exit with its return code."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))


def ranks():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def aggregate(sums, maxes, world, device):
    """Sum `sums` and max `maxes` over ranks (completions / work add up, times take the
    slowest rank): the whole-job numbers rank 0 reports."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(sums) + list(maxes), dtype=torch.float64, device=device)
    if world > 1:
        s, m = t.clone(), t.clone()
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        t = torch.cat([s[:len(sums)], m[len(sums):]])
    vals = t.tolist()
    return vals[:len(sums)], vals[len(sums):]


def cpu_model() -> str:
    """The host CPU model (lscpu's "Model name"), reported with every CPU number."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def bench_config():
    """The workload both arms report (identical dicts, so the driver sees the same config)."""
    from paper_2605_28657_b200.dit import DiTConfig

    dcfg = DiTConfig()
    return {"workload": "config 2: ACE-Step-1.5-shape 24-layer DiT (d=2048, 16/8 heads, SwiGLU 6144, random init), "
                        "60-s latent T=1500 x D=64, ring depth 4, S=8, source present, denoise 1.0, SDE solver; "
                        "one independent stream per GPU",
            "frames": T, "channels": D, "depth": DEPTH, "steps_per_generation": STEPS,
            "dit_params": dcfg.params(), "dit_flops_per_tick": dcfg.flops_per_forward(DEPTH, T),
            "ring_state": "float64", "dit_compute": "bf16 operands, fp32 accumulate / residual stream"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------- clocks -----
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def _query(self):
        try:
            return subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                   "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                  timeout=20).stdout
        except Exception:
            return ""

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
            snap = self._query()  # at least one sample while the GPU is still busy
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


def forward_traffic():
    """DRAM bytes of one DiT forward from the committed ncu launch list (tools/forward_traffic.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_dit_forward_traffic.json")) as fh:
            t = json.load(fh)
        return t["warm"]["dram_bytes"], t["cold"]["dram_bytes"]
    except Exception:
        return None, None


def solve_bytes_per_row(toy: bool):
    # rf_tick_kernel, per element: x read + write (f64), source (f64), sde noise (f64);
    # toy model adds the x0 table, the style offset and the model noise (f64);
    # the DiT path reads the velocity (f32) instead.
    return T * D * ((7 * 8) if toy else (4 * 8 + 4))


def timed_ticks(pipe, steps, flush, stream, phases=False):
    """Device time of `steps` ticks (CUDA events on the pipeline stream around each tick, L2
    flushed before each, outside the events).  phases=True also records the pipeline's
    per-phase events in the same ticks (returned as mean ms per phase), so the roofline's
    model time and `value` come from the same ticks."""
    import torch

    ph = pipe.enable_phase_timing(True) if phases else None
    pairs, completions, launches = [], 0, 0
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        recs = pipe.tick()
        b.record(stream)
        pairs.append((a, b))
        completions += len(recs)
        launches += pipe.launches_last_tick
    torch.cuda.synchronize()
    total = sum(a.elapsed_time(b) for a, b in pairs)
    if phases:
        pipe.enable_phase_timing(False)
        return total, completions, launches, {k: sum(a.elapsed_time(b) for a, b in v) / len(v) for k, v in ph.items()}
    return total, completions, launches


def solve_launch_ms(pipe, flush, iters=40):
    """Device time of the tick's solver launch alone: the last tick's rows re-launched
    through rf_tick_solve, CUDA events on the pipeline stream, inputs evicted from L2 before
    each launch (outside the events).  The in-tick phase events also hold the host's launch
    gap when the GPU waits for the Python tick (the toy path); the flush queued ahead keeps
    the stream busy here, so the events bracket the kernel alone.  Two evictions, both
    timed: "dirty" = the bench's 256-MiB write flush alone (L2 left full of dirty lines the
    solver's reads must write back first: +50-100% at these sizes), "clean" = the write flush
    then a read of the same buffer (the dirty lines written back outside the events; L2 holds
    only clean flush lines, none of the solver's inputs -- ncu's --cache-control all state).
    Returns (clean_ms, dirty_ms).  Advances the ring state (timing only)."""
    import torch

    from paper_2605_28657_b200 import _native

    arr, n = pipe._last_solve
    lib = _native.load()
    T_, D_ = pipe.config.shape
    st = pipe.stream
    res = []
    for clean in (True, False):
        ts = []
        for _ in range(iters):
            with torch.cuda.stream(st):
                flush.fill_(1)
                if clean:
                    torch.amax(flush)   # reads every flush line back (no dirty lines left)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            _native.check(lib.rf_tick_solve(arr, n, T_, D_, pipe.weights.device_offset.data_ptr(), st.cuda_stream),
                          "rf_tick_solve")
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        res.append(sum(a.elapsed_time(b) for a, b in ts) / iters)
    return res[0], res[1]


def decode_240s(codec, world, rank, flush, hbm_peak, iters=10):
    """Config 5: one 240-s latent [6000, 64] decoded sharded over all ranks with halos
    (overlap = receptive field), latent broadcast from rank 0, int16 PCM all-gathered over
    NCCL (sharded_decode.py).  Time = max over ranks of broadcast + shard decode + gather."""
    import torch
    import torch.distributed as dist

    import scenarios
    from paper_2605_28657_b200.sharded_decode import sharded_decode_device

    frames = 6000
    lat = torch.from_numpy(scenarios.keyed(11, "long-latent", (frames, D))).cuda() if rank == 0 else None
    for _ in range(3):
        pcm = sharded_decode_device(codec, lat, src=0, frames=frames)
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pcm = sharded_decode_device(codec, lat, src=0, frames=frames)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = torch.tensor([sorted(ts)[len(ts) // 2]], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    # full-decode check on rank 0 (the sharded PCM must equal the single-GPU full decode)
    exact = None
    if rank == 0:
        exact = bool(torch.equal(pcm, codec.decode_device(lat, 0, frames, 0, True)))
    pcm_bytes = frames * HOP * 2
    lat_bytes = frames * D * 8
    return {"workload": "config 5: 240-s latent [6000, 64] -> 11.52 M int16 samples (48 kHz), sharded "
                        f"decode over {world} GPU(s), halo = receptive field 15 frames, latent broadcast "
                        "+ NCCL all-gather of the PCM inside the timed region",
            "ms": round(ms, 4), "audio_s_per_s": round(240.0 / (ms * 1e-3), 1),
            "bytes_algorithmic": pcm_bytes + lat_bytes,
            "achieved_gbs": round((pcm_bytes + lat_bytes) / (ms * 1e-3) / 1e9, 1), "hbm_peak_gbs": hbm_peak,
            "flops": frames * 344064, "sharded_equals_full_decode": exact}


def config_legs(rf, dit_mod, model, rank, flush, ticks=60):
    """Configs 3 and 4 on the same DiT weights, device time per tick as for
    `value` (events on the pipeline stream, L2 flushed between ticks outside the events).
    config 3: ring depth 8, S=8, one set_denoise per tick from the reference's 60-value
      slider sweep (bench.py:354-357: 1.0 -> 0.5 -> 1.0), so in-flight slots carry
      different baked schedules; 8 DiT rows per tick, one completion per tick.
    config 4: depth 4, request sde_denoise_curve = linspace(0, 1, T) with a source (per-frame
      source blending), and every tick a shared-curve write
      clip(linspace(0, 1, T) * (0.5 + 0.5 sin(2 pi k / 16)), 0, 1) visible from that tick."""
    import numpy as np
    import torch

    sweep = [1.0 - 0.5 * i / 30 for i in range(31)] + [0.5 + 0.5 * j / 29 for j in range(1, 30)]
    out = {}
    m8 = dit_mod.DiT(dit_mod.DiTConfig(), frames=T, max_rows=8, weights=model.weights)
    p3 = rf.StreamPipeline(rf.PipelineConfig(depth=8, steps=STEPS, frames=T, channels=D, seed=rank),
                           request=make_request(rf, rank), velocity_model=dit_mod.DiTVelocity(m8))
    for k in range(4 * STEPS):
        p3.set_denoise(sweep[k % len(sweep)])
        p3.tick()
    torch.cuda.synchronize()
    ev, done, sched = [], 0, set()
    for k in range(ticks):
        p3.set_denoise(sweep[k % len(sweep)])
        with torch.cuda.stream(p3.stream):
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(p3.stream)
        done += len(p3.tick())
        b.record(p3.stream)
        ev.append((a, b))
        sched.update(s.schedule.schedule_id for s in p3._slots if s is not None)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    out["config3"] = {"workload": "depth 8, S=8, 60-s latent, DiT, one set_denoise per tick over the reference's "
                                  "60-value slider sweep (per-slot heterogeneous schedules)",
                      "value": round(done / (ms * 1e-3), 3), "unit": UNIT, "ms_per_step": round(ms / ticks, 4),
                      "ticks": ticks, "completions": done, "distinct_schedules_in_flight": len(sched)}
    del p3, m8
    torch.cuda.empty_cache()

    lin = np.linspace(0.0, 1.0, T)
    req = make_request(rf, rank)
    req4 = rf.GenerationRequest(conditions=req.conditions, curves=rf.CurveSet(sde_denoise_curve=lin))
    p4 = rf.StreamPipeline(rf.PipelineConfig(depth=DEPTH, steps=STEPS, frames=T, channels=D, seed=rank),
                           request=req4, velocity_model=dit_mod.DiTVelocity(model))
    shared = lambda k: np.clip(lin * (0.5 + 0.5 * np.sin(2 * np.pi * k / 16)), 0.0, 1.0)  # noqa: E731
    for k in range(4 * STEPS):
        p4.set_shared_curve("sde_denoise_curve", shared(k))
        p4.tick()
    torch.cuda.synchronize()
    ev, done = [], 0
    for k in range(ticks):
        p4.set_shared_curve("sde_denoise_curve", shared(k))   # host -> device, visible from this tick
        with torch.cuda.stream(p4.stream):
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(p4.stream)
        done += len(p4.tick())
        b.record(p4.stream)
        ev.append((a, b))
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    out["config4"] = {"workload": "depth 4, S=8, 60-s latent, DiT, request sde_denoise_curve = linspace(0,1,T) "
                                  "with source (per-frame blend), a shared-curve write every tick",
                      "value": round(done / (ms * 1e-3), 3), "unit": UNIT, "ms_per_step": round(ms / ticks, 4),
                      "ticks": ticks, "completions": done}
    del p4
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_28657_b200 as rf
    from paper_2605_28657_b200 import dit as dit_mod

    world, rank, local = ranks()
    if torch.cuda.device_count() < local + 1:
        sys.exit(f"bench.py: rank {rank} needs cuda:{local} but only {torch.cuda.device_count()} GPU(s) are visible")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    hbm_peak, bf16_burst, bf16_sust, peak_src = peaks()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    conf = rf.PipelineConfig(depth=DEPTH, steps=STEPS, frames=T, channels=D, seed=rank)

    # ---------------- config 2: the DiT velocity model ----------------
    dcfg = dit_mod.DiTConfig()
    model = dit_mod.DiT(dcfg, frames=T, max_rows=DEPTH)
    pipe = rf.StreamPipeline(conf, request=make_request(rf, rank), velocity_model=dit_mod.DiTVelocity(model))
    st = pipe.stream
    # setup: fill the ring (warmup pacing admits one slot per ceil(S/D) ticks) until the first
    # generation completes -- the steady state every timed tick is in; then W warm-up ticks
    fill = 0
    while fill < 4 * STEPS and not pipe.tick():
        fill += 1
    for _ in range(args.warmup):
        pipe.tick()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        dev_ms, completions, launches, phase_ms = timed_ticks(pipe, args.steps, flush, st, phases=True)
    clocks = clk.summary()
    dit_flops = dcfg.flops_per_forward(DEPTH, T)
    dit_tflops = dit_flops / (phase_ms["model"] * 1e-3) / 1e12

    # ---- end-to-end through the public API with host buffers ----
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    curve = np.linspace(0.0, 1.0, T)
    codec = rf.ToyCodec(channels=D, hop=HOP)
    gate = rf.GatedDecoder(codec, window_frames=WINDOW, overlap=OVERLAP)
    t0 = time.perf_counter()
    e2e_done, h2d, d2h = 0, 0, 0
    for k in range(args.steps):
        # a control write every tick whose value flips every 8 ticks, so the similarity filter
        # sees both settled and changing completions
        pipe.set_shared_curve("sde_denoise_curve", curve if (k // 8) % 2 else 1.0)   # host -> device, [T] f64
        h2d += T * 8
        for r in pipe.tick():
            _ = r.latent                                                       # device -> host, [T, D] f64
            d2h += T * D * 8
            gate.feed(r)                                                       # gated 3-s window decode
            d2h += gate.latest_pcm().samples.nbytes                            # device -> host, int16 PCM
            e2e_done += 1
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    gated = {"window_frames": WINDOW, "overlap": OVERLAP, "decodes": gate.decodes, "skips": gate.skips,
             "skip_rate": round(gate.skip_rate, 3),
             "note": "similarity-filter-gated decode (PAPER.md:203): flagged completions reuse the last chunk"}
    pipe.set_shared_curve("sde_denoise_curve", 1.0)

    # ---- windowed decode (3-s window + overlap 15) of the last completion ----
    configs = None if args.no_configs else config_legs(rf, dit_mod, model, rank, flush)
    lat = pipe._last_emitted
    with torch.cuda.stream(st):
        for _ in range(3):
            codec.decode_device(lat, T - WINDOW, T, OVERLAP, False)
        # the latent and the packed weights evicted from L2 before each decode (outside the
        # events) two ways: the write flush alone leaves ~126 MB of dirty lines whose
        # write-back the decode's first DRAM reads queue behind (a constant ~22.5 us whatever
        # the kernel, tools/decode_window_time.py); the write flush + a read-back of the same
        # buffer leaves clean lines only (ncu's cache-control state) -- reported as the value
        ev = {True: [], False: []}
        for clean in (True, False):
            for _ in range(10):
                flush.fill_(1)
                if clean:
                    torch.amax(flush)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                codec.decode_device(lat, T - WINDOW, T, OVERLAP, False)
                b.record(st)
                ev[clean].append((a, b))
    torch.cuda.synchronize()
    decode_ms = sorted(a.elapsed_time(b) for a, b in ev[True])[5]
    decode_dirty_ms = sorted(a.elapsed_time(b) for a, b in ev[False])[5]
    weights_keep = model.weights
    del pipe, model
    torch.cuda.empty_cache()

    long_decode = decode_240s(codec, world, rank, flush, hbm_peak)

    # ---- the same DiT forward written with library kernels (cuBLAS GEMMs + SDPA) ----
    library = None
    if not args.no_library_baseline and rank == 0:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import dit_torch_baseline

        library = dit_torch_baseline.compare(rows=DEPTH, check=False)
        library["what"] = ("config-2 DiT forward (4 rows) in stock PyTorch: cuBLAS bf16 GEMMs, SDPA attention, "
                           "torch elementwise norms/RoPE/SwiGLU, one CUDA graph (tools/dit_torch_baseline.py); "
                           "native = this repo's tcgen05 forward on the same weights")

    # ---------------- config 5 generation: the DiT tick at 240 s ----------------
    dit240 = None if args.no_240s_dit else dit_tick_240s(rf, dit_mod, weights_keep, rank, flush, bf16_sust)
    del weights_keep
    torch.cuda.empty_cache()

    # ---------------- toy-velocity leg (the reference's own model) ----------------
    toy = None
    if not args.no_toy:
        tp = rf.StreamPipeline(conf, request=make_request(rf, rank))
        for _ in range(32):
            tp.tick()
        torch.cuda.synchronize()
        t_ms, t_done, t_launch = timed_ticks(tp, 64, flush, tp.stream)
        # phases from separate ticks: at ~0.13 ms per tick the phase events would be a
        # visible part of the timed region
        t_phase = timed_ticks(tp, 16, flush, tp.stream, phases=True)[3]
        sb = DEPTH * solve_bytes_per_row(True)
        # host-inclusive rate: ticks back to back (no flush), wall clock
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        w_done = sum(len(tp.tick()) for _ in range(256))
        torch.cuda.synchronize()
        w_s = time.perf_counter() - w0
        nc = tp.noise_cache
        cache_stats = {"hits": nc.hits, "misses": nc.misses, "resident_bytes": nc.bytes}
        solve_ms, solve_dirty_ms = solve_launch_ms(tp, flush)   # last: it advances the ring
        del tp
        # the same leg with the noise cache off (every draw regenerated every tick)
        tq = rf.StreamPipeline(conf, request=make_request(rf, rank), noise_cache_bytes=0)
        for _ in range(32):
            tq.tick()
        torch.cuda.synchronize()
        q_ms, q_done, _ = timed_ticks(tq, 64, flush, tq.stream)
        del tq
        toy = {"value": round(t_done / (t_ms * 1e-3), 2), "unit": UNIT, "ms_per_step": round(t_ms / 64, 5),
               "wall": {"value": round(w_done / w_s, 1), "unit": UNIT, "us_per_tick": round(w_s / 256 * 1e6, 1),
                        "note": "256 ticks back to back, wall clock (host Python + device), no L2 flush"},
               "noise_cache": dict(cache_stats, note="device cache of keyed draws (seed, content key, step, tag); "
                                   "steady state regenerates nothing"),
               "noise_cache_off": {"value": round(q_done / (q_ms * 1e-3), 2), "ms_per_step": round(q_ms / 64, 5)},
               "phase_ms": {k: round(v, 5) for k, v in t_phase.items()},
               "solver_roofline": {"bound": "hbm", "kernel": "rf_tick_fast_kernel",
                                   "achieved": round(sb / (solve_ms * 1e-3) / 1e9, 1), "peak": hbm_peak,
                                   "unit": "GB/s", "frac": round(sb / (solve_ms * 1e-3) / 1e9 / hbm_peak, 4),
                                   "launch_us": round(solve_ms * 1e3, 2),
                                   "launch_us_behind_dirty_flush": round(solve_dirty_ms * 1e3, 2),
                                   "algorithmic_bytes_per_launch": sb,
                                   "note": "the tick's solver launch re-issued 40x with its inputs evicted from L2 "
                                           "(write flush + read-back: clean L2, as ncu's cache control), CUDA events "
                                           "on the pipeline stream (bench.solve_launch_ms); behind the write flush "
                                           "alone the solver first writes back ~126 MB of dirty flush lines; "
                                           "phase_ms.solve also holds the host's launch gap"},
               "gpu_launches": t_launch, "dtype": "f64",
               "note": "same ring and solver with ToyFlowModel velocities (bit-exact vs the reference)"}

    # ---- aggregate over ranks (sums of work, max of times) ----
    (completions_all, e2e_all, flops_all, launches_all), (dev_ms_max, e2e_max, model_ms_max) = aggregate(
        [completions, e2e_done, dit_flops * args.steps, launches],
        [dev_ms, e2e_s, phase_ms["model"] * args.steps], world, dev)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    value = completions_all / (dev_ms_max * 1e-3)
    # whole-job tensor throughput of the forwards against world x the sustained peak
    agg_tflops = flops_all / (model_ms_max * 1e-3) / 1e12
    traffic_warm, traffic_cold = forward_traffic()
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dev_ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded latents, random-init DiT)",
        "config": bench_config(),
        "l2": "flushed (256 MiB write) between timed ticks, outside the events",
        "completions_timed": int(completions_all),
        "e2e": {"value": round(e2e_all / e2e_max, 3), "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps,
                "note": "wall clock through StreamPipeline: a host shared-curve write every tick (value flips every 8), "
                        "every CompletionRecord.latent read back to host, its 3-s playback window decoded "
                        "through GatedDecoder and the int16 PCM read back to host",
                "gated_decode": gated},
        "windowed_decode_ms": round(decode_ms, 5),
        "windowed_decode_ms_behind_dirty_flush": round(decode_dirty_ms, 5),
        "decode_240s": long_decode,
        "phase_ms": {k: round(v, 4) for k, v in phase_ms.items()},
        "roofline": {"bound": "tensor", "kernel": "dit_forward (tcgen05 GEMMs + attention + norms, one launch set)",
                     "achieved": round(agg_tflops, 1), "peak": round(world * bf16_sust, 1), "unit": "TFLOP/s",
                     "frac": round(agg_tflops / (world * bf16_sust), 4), "traffic": traffic_warm,
                     "traffic_note": "DRAM read+write bytes of one forward (sum over its launches) from the "
                                     "committed ncu launch list profiles/r2_dit_forward_traffic.json, "
                                     f"--cache-control none; cold-cache sum {traffic_cold}",
                     "algorithmic_flops_per_launch": dit_flops,
                     "peak_source": f"{peak_src} bf16 sustained x {world} GPU(s) (burst {bf16_burst} per GPU)",
                     "per_gpu_frac": round(agg_tflops / world / bf16_sust, 4)},
        "gpu_launches": int(launches_all),
        "clocks": clocks,
    }
    if toy is not None:
        line["toy_path"] = toy
    if library is not None:
        line["library_baseline"] = library
    if configs is not None:
        line["other_configs"] = configs
    if dit240 is not None:
        line["config5_dit_tick"] = dit240
    if not args.no_cpu_baseline:
        # the same workload (config 2 with the DiT) on the box's host cores, bounded sample
        line["cpu_baseline"] = cpu_dit_baseline(args.cpu_seconds, os.cpu_count() or 1)
        # and the reference's own toy model on one core (its CPU speed on its only model)
        line["cpu_baseline_toy_model"] = cpu_baseline(args.cpu_seconds, processes=1)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def dit_tick_240s(rf, dit_mod, weights, rank, flush, bf16_sust, ticks=16):
    """Config 5's generation side: the DiT tick on a 240-s latent (T=6000 -> 3000 tokens),
    depth 4, S=8, same weights; device time per tick as for `value` (PAPER.md:322 quotes
    the production decoder at B=8 for this length)."""
    import torch

    frames = 6000
    m = dit_mod.DiT(dit_mod.DiTConfig(), frames=frames, max_rows=DEPTH, weights=weights)
    import scenarios

    src = scenarios.keyed(rank, "bench-source-240", (frames, D))
    req = rf.GenerationRequest(conditions=(rf.ConditionSet(prompt_hash=rf.content_hash("bench", "bench prompt"),
                                                           source=src),))
    p = rf.StreamPipeline(rf.PipelineConfig(depth=DEPTH, steps=STEPS, frames=frames, channels=D, seed=rank),
                          request=req, velocity_model=dit_mod.DiTVelocity(m))
    fill = 0
    while fill < 4 * STEPS and not p.tick():
        fill += 1
    for _ in range(3):
        p.tick()
    torch.cuda.synchronize()
    ms, done, _, ph = timed_ticks(p, ticks, flush, p.stream, phases=True)
    flops = dit_mod.DiTConfig().flops_per_forward(DEPTH, frames)
    tf = flops / (ph["model"] * 1e-3) / 1e12
    solve_ms, solve_dirty_ms = solve_launch_ms(p, flush)   # last: it advances the ring
    sb = DEPTH * frames * D * (4 * 8 + 4)  # solve_bytes_per_row(False) at T = 6000
    hbm_peak = peaks()[0]
    del p, m
    torch.cuda.empty_cache()
    return {"workload": "config 5 generation: 240-s latent T=6000 x D=64 (3000 DiT tokens), depth 4, S=8, DiT",
            "value": round(done / (ms * 1e-3), 3), "unit": UNIT, "ms_per_step": round(ms / ticks, 3),
            "ticks": ticks, "completions": done, "phase_ms": {k: round(v, 3) for k, v in ph.items()},
            "dit_flops_per_tick": flops, "dit_tflops": round(tf, 1), "frac_of_sustained_peak": round(tf / bf16_sust, 4),
            "solver_roofline": {"bound": "hbm", "kernel": "rf_tick_fast_kernel", "launch_us": round(solve_ms * 1e3, 2),
                                "launch_us_behind_dirty_flush": round(solve_dirty_ms * 1e3, 2),
                                "achieved": round(sb / (solve_ms * 1e-3) / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
                                "frac": round(sb / (solve_ms * 1e-3) / 1e9 / hbm_peak, 4),
                                "algorithmic_bytes_per_launch": sb,
                                "note": "DiT rows: x read + write, source, SDE noise (f64), velocity (f32); "
                                        "bench.solve_launch_ms"}}


def run_stub(args):
    """Harness test on the CPU: the torchrun launch, rank setup, aggregation and JSON line
    of the real arm over gloo with a stub workload (each rank 'completes' one generation
    every other step).  Never a bench number: impl 'stub'."""
    import torch
    import torch.distributed as dist

    world, rank, _ = ranks()
    if world > 1:
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    done = 0
    for k in range(args.warmup + args.steps):
        if k >= args.warmup and k % 2:
            done += 1
    wall_ms = (time.perf_counter() - t0) * 1e3 + 1e-3
    (done_all, ranks_seen), (ms_max,) = aggregate([done, 1], [wall_ms], world, torch.device("cpu"))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "impl": "stub", "value": done_all / (ms_max * 1e-3), "unit": UNIT,
                          "n_gpus": world, "ranks_reporting": int(ranks_seen), "completions_timed": int(done_all),
                          "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                          "data": "stub workload on CPU/gloo: harness test only, not a measurement"}), flush=True)
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
    return {"value": round(done / wall, 3), "unit": UNIT, "cores": processes, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"oracle/ringflow_np.py StreamPipeline restatement (toy velocity model, the reference's "
                      f"only model), config-2 shape (T=1500, D=64, depth 4, S=8), {processes} independent "
                      f"stream(s), {ticks} warm ticks after {4 * STEPS} warmup, {wall:.1f} s wall, float64 numpy, "
                      f"1 thread/process"}


def cpu_dit_baseline(seconds, threads, max_ticks=None):
    """Config 2 on the host CPU: the reference's tick (oracle/ringflow_np.py, float64 numpy)
    with the DiT in its model slot (oracle/dit_fp32.py: the same network with bf16 GEMM and
    attention operands -- the precision of the GPU arm and the CPU's fastest path (AMX) --
    torch on all `threads` host threads; one forward per ring row per tick).  The ring is filled with the
    toy model first (cheap), then steady-state DiT ticks are timed: at least one, then until
    `seconds` or `max_ticks`.  completions/s = row-steps / S / wall (every completion is S
    row-steps; at depth 4 one completes every other tick)."""
    import torch

    import scenarios

    import oracle.ringflow_np as O
    from oracle.dit_fp32 import CpuDiTVelocity
    from paper_2605_28657_b200.dit import DiTConfig

    torch.set_num_threads(threads)
    src = scenarios.keyed(0, "bench-source", (T, D))
    req = O.Request([O.Cond(O.chash("bench", "bench prompt"), source=src)])
    pipe = O.Pipeline(depth=DEPTH, steps=STEPS, frames=T, channels=D, seed=0, request=req)
    for _ in range(4 * STEPS):
        pipe.tick()
    pipe.model = CpuDiTVelocity(DiTConfig(), T, bf16=True)   # the fastest CPU path (bf16 AMX GEMMs)
    pipe.tick()   # untimed: first-touch of the fp32 weights
    row_steps, ticks = 0, 0
    t0 = time.perf_counter()
    while ticks == 0 or (time.perf_counter() - t0 < seconds and (max_ticks is None or ticks < max_ticks)):
        row_steps += sum(1 for s in pipe.slots if s is not None)
        pipe.tick()
        ticks += 1
    wall = time.perf_counter() - t0
    return {"value": round(row_steps / STEPS / wall, 5), "unit": UNIT, "cores": threads, "kind": "port",
            "cpu_model": cpu_model(), "ticks": ticks,
            "sample": f"config 2 on the host CPU: oracle/ringflow_np.py tick (the reference's algorithm, float64 "
                      f"numpy) with the ACE-Step-shape DiT (oracle/dit_fp32.py, torch CPU, bf16 GEMM/attention "
                      f"operands with fp32 accumulation, {threads} threads) in "
                      f"the model slot; {ticks} steady-state tick(s) ({row_steps} DiT row forwards + SDE steps) "
                      f"in {wall:.1f} s after the ring was filled; completions/s = row-steps / S / wall; "
                      f"one DiT forward per ring row per tick (the reference's per-slot model loop, "
                      f"pipeline.py:449-464), rows not batched"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    # each step = one steady-state config-2 tick on the CPU; bounded to ~90 s of ticks
    base = cpu_dit_baseline(90.0, procs, max_ticks=args.steps)
    toy = cpu_baseline(10.0, processes=procs)
    line = {
        "metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": base["ticks"], "steps_requested": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded latents, random-init DiT)",
        "impl": "reference",
        "config": bench_config(),
        "arm": "the reference's tick on the host CPU (oracle port, float64 numpy) with the DiT (torch CPU, bf16 "
               "operands, all host threads) in its model slot",
        "cpu_baseline": base,
        "toy_model": {**toy, "note": "the reference's own ToyFlowModel at config-2 shape, one stream per host "
                                     "core: the reference's CPU speed on its only model"},
        "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def refuse_tuning_env():
    """The product library reads no environment knobs; refuse to time a run that sets RF_*
    variables anyway (a leftover from an experiment must not leak into a bench number)."""
    bad = sorted(k for k in os.environ if k.startswith("RF_"))
    if bad:
        sys.exit(f"bench.py: refusing to run with RF_* environment variables set: {bad}")


if __name__ == "__main__":
    refuse_tuning_env()
    a = parse()
    maybe_respawn(a)
    if a.impl == "reference":
        run_reference(a)
    elif a.stub:
        run_stub(a)
    else:
        run_ours(a)
