"""Sustained DiT forward rate: 2 s of back-to-back graph replays (config 2, 4 rows) after a
1 s warm-up, median over 20 groups of 10 -- the board-power-capped steady state the tick runs
in (short runs read a few % faster on a cool GPU).  Also reports the SM clock and the board
energy per forward (NVML total-energy counter) over the timed groups: at the power cap the
forward's time is set by its energy, so this is the number a design change has to lower."""
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402


def _nvml():
    try:
        import pynvml

        pynvml.nvmlInit()
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:  # noqa: BLE001
        return None, None


def main():
    torch.cuda.set_stream(torch.cuda.Stream())
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    cfg = D.DiTConfig()
    dit = D.DiT(cfg, frames=1500, max_rows=max(rows, 4))
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(rows)]
    ts = [1.0 - 0.1 * i for i in range(rows)]
    conds = [dit.cond_tokens(i) for i in range(rows)]
    t0 = time.time()
    while time.time() - t0 < 1.0:
        dit.forward(xs, ts, conds)
    torch.cuda.synchronize()
    nv, h = _nvml()
    clocks, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            clocks.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            time.sleep(0.05)

    th = None
    e0 = None
    if nv:
        e0 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        th = threading.Thread(target=sample, daemon=True)
        th.start()
    res = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            dit.forward(xs, ts, conds)
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 10)
    extra = ""
    if nv:
        e1 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        stop.set()
        th.join()
        extra = f"  sm {statistics.median(clocks):.0f} MHz  {(e1 - e0) / 200:.0f} mJ/forward"
    ms = statistics.median(res)
    print(f"sustained forward {ms:.3f} ms  {cfg.flops_per_forward(rows, 1500) / ms / 1e9:.1f} TFLOP/s "
          f"(min {min(res):.3f} max {max(res):.3f}){extra}")


if __name__ == "__main__":
    main()
