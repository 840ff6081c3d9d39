"""Hot instructions of one kernel in an ncu --set full report: top warp-stall-sampled SASS
lines with their CUDA source line (needs -lineinfo), plus headline metrics.

    python tools/ncu_hot.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "launch__registers_per_thread"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, v = raw[0], raw[2] if len(raw) > 2 else raw[1]
    for i, n in enumerate(h):
        if n in METRICS:
            print(f"{n:70s} {v[i]}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass,cuda"])))
               if False else csv.reader(io.StringIO(run([rep, "--page", "source", "--csv"]))))
    hdr = src[1]
    si, ti = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    rows = [(int(r[si]), r[ti].strip()) for r in src[2:] if len(r) > si and r[si].isdigit()]
    tot = sum(a for a, _ in rows)
    print(f"stall samples: {tot}")
    idx = sorted(range(len(rows)), key=lambda i: -rows[i][0])[:top]
    for i in sorted(idx):
        print(f"{i:5d} {rows[i][0]:6d} {100 * rows[i][0] / tot:5.1f}%  {rows[i][1][:90]}")


if __name__ == "__main__":
    main()
