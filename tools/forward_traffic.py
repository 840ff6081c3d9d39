"""Per-forward DRAM traffic and kernel time of the DiT from ncu launch lists
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum), one with
the default cache control (caches flushed before every kernel: cold) and one with
--cache-control none (warm, as in the real forward).  Writes the JSON bench.py reads for
roofline.traffic.

    python tools/forward_traffic.py cold.csv warm.csv out.json"""
import csv
import json
import sys
from collections import defaultdict


def forwards(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3,
             "ms": 1e3, "msecond": 1e3}
    launches = defaultdict(dict)
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        d = launches[int(r[0])]
        d["name"] = r[ki].split("(")[0]
        d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    seq = [launches[i] for i in sorted(launches)]
    groups, cur = [], None
    for d in seq:
        if "rf_dit_set_rows" in d["name"]:
            cur = []
            groups.append(cur)
        if cur is not None:
            cur.append(d)
    return [g for g in groups if any("rf_gemm_kernel" in d["name"] for d in g)]


def summarize(path):
    fw = forwards(path)
    g = fw[-2] if len(fw) > 1 else fw[-1]   # a complete forward (the last may be cut by -c)
    return {"launches": len(g), "kernel_time_sum_us": round(sum(d.get("gpu__time_duration.sum", 0) for d in g), 1),
            "dram_read_bytes": int(sum(d.get("dram__bytes_read.sum", 0) for d in g)),
            "dram_write_bytes": int(sum(d.get("dram__bytes_write.sum", 0) for d in g))}


def main():
    cold, warm, out = sys.argv[1:4]
    res = {"what": "one config-2 DiT forward (4 rows x 750 tokens), sums over its kernel launches",
           "cold": summarize(cold), "warm": summarize(warm),
           "commands": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                       "--clock-control none [--cache-control none] python tools/dit_check.py 4 --no-ref"}
    for k in ("cold", "warm"):
        res[k]["dram_bytes"] = res[k]["dram_read_bytes"] + res[k]["dram_write_bytes"]
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
