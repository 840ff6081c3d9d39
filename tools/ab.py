"""A/B timing of the config-2 DiT forward (CUDA graph replay) under different environment
settings, alternated in fresh processes: python tools/ab.py "A=1" "A=0 B=2" ... [--rounds N]"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(envs):
    env = dict(os.environ)
    for kv in envs.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "dit_check.py"), "4", "--no-ref", "--graph"],
                         env=env, capture_output=True, text=True, timeout=300).stdout
    m = re.search(r"graph forward ([0-9.]+) ms", out)
    return float(m.group(1)) if m else float("nan")


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--rounds")]
    rounds = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--rounds=")), "4"))
    res = {a: [] for a in args}
    for _ in range(rounds):
        for a in args:
            res[a].append(run(a))
    for a in args:
        v = sorted(res[a])
        print(f"{a!r:40s} median {v[len(v) // 2]:.3f} ms  all {' '.join(f'{x:.3f}' for x in res[a])}", flush=True)


if __name__ == "__main__":
    main()
