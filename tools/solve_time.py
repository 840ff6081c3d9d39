"""Device time of the config-2 toy tick's solver launch (bench.solve_launch_ms) and its HBM
rate; run under ncu (-k regex:rf_tick) for the kernel's own duration and DRAM bytes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_28657_b200 as rf  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
frames = int(sys.argv[2]) if len(sys.argv) > 2 else bench.T
bench.T = frames
conf = rf.PipelineConfig(depth=bench.DEPTH, steps=bench.STEPS, frames=frames, channels=bench.D, seed=0)
dit = "dit" in sys.argv[3:]
if dit:   # DiT rows (fp32 velocities from the DiT output), the full config-2 network
    from paper_2605_28657_b200 import dit as dit_mod
    vm = dit_mod.DiTVelocity(dit_mod.DiT(dit_mod.DiTConfig(), frames=frames, max_rows=bench.DEPTH))
    p = rf.StreamPipeline(conf, request=bench.make_request(rf, 0), velocity_model=vm)
else:
    p = rf.StreamPipeline(conf, request=bench.make_request(rf, 0))
for _ in range(32):
    p.tick()
torch.cuda.synchronize()
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
ms, dirty = bench.solve_launch_ms(p, flush, iters)
sb = bench.DEPTH * bench.solve_bytes_per_row(not dit)
hbm = bench.peaks()[0]
print(f"T={frames} {'dit' if dit else 'toy'}: solve launch {ms * 1e3:.2f} us  {sb / ms / 1e6:.1f} GB/s  frac {sb / ms / 1e6 / hbm:.3f}  (behind the dirty flush {dirty * 1e3:.2f} us)")
