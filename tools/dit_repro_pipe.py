"""Reproducibility probe on the ring's real DiT inputs: stream config 2 for a few ticks,
record every forward's inputs, then replay each recorded forward twice per attention
variant and report the calls whose outputs differ between replays."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import scenarios  # noqa: E402

import paper_2605_28657_b200 as rf  # noqa: E402
from paper_2605_28657_b200 import _native, dit as D  # noqa: E402


def main():
    lib = _native.load()
    T, Dc = 1500, 64
    src = scenarios.keyed(0, "bench-source", (T, Dc))
    req = rf.GenerationRequest(conditions=(rf.ConditionSet(prompt_hash=rf.content_hash("bench", "bench prompt"),
                                                           source=src),))
    conf = rf.PipelineConfig(depth=4, steps=8, frames=T, channels=Dc, seed=0)
    dit = D.DiT(D.DiTConfig(), frames=T, max_rows=4)
    rec = []
    orig = dit.forward

    def recording(xs, ts, conds, out=None):
        rec.append(([x.clone() for x in xs], list(ts), list(conds)))
        return orig(xs, ts, conds, out)

    dit.forward = recording
    pipe = rf.StreamPipeline(conf, request=req, velocity_model=D.DiTVelocity(dit))
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
        pipe.tick()
    torch.cuda.synchronize()
    dit.forward = orig
    print(f"recorded {len(rec)} forwards, rows {[len(r[0]) for r in rec]}", flush=True)
    for v in [tuple(int(y) for y in x.split(":")) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0:0", "1:0", "3:0"])]:
        lib.rf_attn_set_variant(*v)
        d2 = D.DiT(D.DiTConfig(), frames=T, max_rows=4, weights=dit.weights)
        bad = []
        for i, (xs, ts, conds) in enumerate(rec):
            a = d2.forward(xs, ts, conds).clone()
            b = d2.forward(xs, ts, conds).clone()
            if not torch.equal(a, b):
                bad.append((i, len(xs), f"{(a - b).abs().max().item():.2e}"))
        print(f"variant {v}: {len(bad)} of {len(rec)} forwards differ between replays: {bad[:8]}", flush=True)
        del d2
    lib.rf_attn_set_variant(-1, -1)


if __name__ == "__main__":
    main()
