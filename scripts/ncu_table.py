"""Per-launch table of an ncu --set full capture (run here on the .ncu-rep gpurun brings back):
python scripts/ncu_table.py <capture.ncu-rep>... > profiles/<tag>.md

Columns: duration, DRAM read/write, achieved DRAM GB/s, FP64 pipe (% of peak, active
cycles), issue active, occupancy, registers, grid; then totals over the listed launches."""
import csv
import io
import os
import subprocess
import sys

COLS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB"),
    ("dram__bytes_write.sum", "MB"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
    ("launch__registers_per_thread", ""),
    ("launch__grid_size", ""),
]
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    return name.replace("void ", "").split("(")[0]


def main():
    for rep in sys.argv[1:]:
        hdr, units, data = rows(rep)
        print(f"### {os.path.basename(rep)}\n")
        print("| kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s | FP64 pipe % | issue % | occupancy % "
              "| regs | grid |\n|---|---|---|---|---|---|---|---|---|---|")
        tot_us = tot_r = tot_w = 0.0
        fp_w = 0.0
        for row in data:
            v = {}
            for key, unit in COLS:
                i = hdr.index(key)
                x = float(row[i].replace(",", "")) if row[i] else 0.0
                v[key] = x * SCALE.get(units[i], 1.0) if unit in ("us", "MB") else x
            us, rd, wr = v["gpu__time_duration.sum"], v["dram__bytes_read.sum"], v["dram__bytes_write.sum"]
            fp = v["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
            tot_us += us
            tot_r += rd
            tot_w += wr
            fp_w += fp * us
            print(f"| `{short(row[hdr.index('Kernel Name')])}` | {us:.1f} | {rd:.1f} | {wr:.1f} | "
                  f"{(rd + wr) / us * 1e3:.0f} | {fp:.1f} | "
                  f"{v['smsp__issue_active.avg.pct_of_peak_sustained_active']:.1f} | "
                  f"{v['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | "
                  f"{int(v['launch__registers_per_thread'])} | {int(v['launch__grid_size'])} |")
        if tot_us:
            print(f"| **total** | {tot_us:.1f} | {tot_r:.1f} | {tot_w:.1f} | {(tot_r + tot_w) / tot_us * 1e3:.0f} | "
                  f"{fp_w / tot_us:.1f} (time-weighted) | | | | |\n")


if __name__ == "__main__":
    main()
