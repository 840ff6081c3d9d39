"""Per-kernel summary of the last DiT forward in an ncu launch list (tools/fwd_check.sh)."""
import csv
import sys
from collections import defaultdict


def main(path, last=231):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launch = {}
    for r in rows[start + 1:]:
        if len(r) > vi:
            launch.setdefault(r[ii], {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    seq = list(launch.values())[-last:]
    agg = defaultdict(list)
    for d in seq:
        agg[d["k"].split("(")[0][:60]].append(d["gpu__time_duration.sum"])
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:60s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:8.2f} us share={sum(v) / tot * 100:5.1f}%")
    print(f"sum of {len(seq)} launches: {tot / 1e6:.3f} ms (cold, serialised)")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 231)
