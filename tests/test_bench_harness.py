"""bench.py's multi-rank launch and aggregation on the CPU (gloo, world 2), stub workload.

``python bench.py --gpus 2 --stub`` must start two ranks itself (re-executing under
torch.distributed.run when no torchrun environment is present), aggregate over both
(sum of completions, max of times) and print one JSON line from rank 0 with n_gpus = 2.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                           "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=300, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(x) for x in res.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1, res.stdout   # rank 0 alone prints
    return lines[0]


@pytest.mark.parametrize("n", [1, 2])
def test_bench_spawns_ranks_and_aggregates(n):
    line = _run("--gpus", str(n), "--stub", "--steps", "6", "--warmup", "3")
    assert line["impl"] == "stub" and line["n_gpus"] == n and line["ranks_reporting"] == n
    assert line["completions_timed"] == 3 * n      # every rank's 3 completions summed
    assert line["value"] > 0 and line["scaling"] == "weak"


def test_bench_refuses_tuning_env():
    env = dict(os.environ, RF_SOME_KNOB="1")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--stub"], capture_output=True, text=True,
                         timeout=120, cwd=ROOT, env=env)
    assert res.returncode != 0 and "RF_" in res.stderr
