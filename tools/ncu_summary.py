"""Key metrics of ncu --set full captures (.ncu-rep), one block per kernel launch.

    python tools/ncu_summary.py report.ncu-rep [...] > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

UNIT = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0,
        "nsecond": 1e-3, "msecond": 1e3}
KEYS = [
    ("gpu__time_duration.sum", "duration (us)", None),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (GHz)", 1),
    ("dram__bytes_read.sum", "DRAM read (MB)", None),
    ("dram__bytes_write.sum", "DRAM write (MB)", None),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)", 1),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput (% of peak)", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (% of elapsed)", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (% of active)", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (%)", 1),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem->tensor wavefronts (%)", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (%)", 1),
    ("launch__registers_per_thread", "registers/thread", 1),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA (KB)", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
]


def main():
    for path in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            print(f"== {path.split('/')[-1]}: {d.get('Kernel Name', '')[:110]}")
            for k, label, scale in KEYS:
                v = d.get(k)
                if v in (None, ""):
                    continue
                try:
                    unit = u.get(k, "")
                    x = float(v.replace(",", "")) * (UNIT.get(unit, 1.0) if scale is None else scale)
                    print(f"  {label:38s} {x:12.3f}   [{k} {unit}]")
                except ValueError:
                    print(f"  {label:38s} {v}")
            print()


if __name__ == "__main__":
    main()
