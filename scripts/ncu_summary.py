"""Summarise ncu captures for profiles/ (run here, on the .ncu-rep / CSV brought back by gpurun).

python scripts/ncu_summary.py <tag> <launches.csv> <kernel.ncu-rep>... > profiles/<tag>.md
Also updates profiles/traffic.json with DRAM bytes per launch of the near-field evaluation
(k_neval) and k_far."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (of active cycles)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "FP64 pipe active % (of elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp-instruction"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-instructions"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread-instructions"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "L1 hit rate (global loads) %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle / issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * mult


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
        name = name.split("(")[0]
        if "<" in name:
            name = name[:name.index("<")] + "<" + name[name.index("<") + 1:].split(">")[0] + ">"
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    return tot, cnt


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    cfg = os.environ.get("NCU_CFG", "cfg1")  # which BASELINE configuration the captures ran
    desc = {"cfg1": "cfg1 (N=1M cube, p=8, theta=0.5, N0=2000)",
            "cfg2": "cfg2 (N=4M sphere, p=10, theta=0.7, N0=2000)",
            "cfg3": "cfg3 (N=16M cube, p=8, theta=0.5, N0=4000)",
            "cfg4": "cfg4 (8M Gaussian-mixture sources, 8M uniform targets, p=8, theta=0.6, N0=2000)"}[cfg]
    print(f"# ncu summary — {tag}\n")
    print("Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
          f"(sm_100a), one launch per kernel, BASELINE {desc}. "
          "ncu times are cold-cache and serialised: compare shares, not absolutes.\n")
    tot, cnt = launches(lcsv)
    # a bench.py launch list also holds its live FP64 peak probe (not part of a step) and
    # warm-up + timed steps: report per step, counting steps by near-field launches
    probe = [k for k in tot if "fp64_peak" in k]
    for k in probe:
        tot.pop(k)
        cnt.pop(k)
    steps = max([c for k, c in cnt.items() if k.startswith("st::k_neval")] or [1])
    T = sum(tot.values()) / steps
    title = "one treecode step" if steps == 1 else f"per treecode step (list of {steps} steps" + \
        (", FP64 peak probe excluded)" if probe else ")")
    print(f"## Launch list (`--metrics gpu__time_duration.sum`), {title}\n")
    print("| kernel | launches/step | ms/step | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:14]:
        print(f"| `{k}` | {cnt[k] / steps:g} | {v / steps:.3f} | {100 * v / steps / T:.1f}% |")
    print(f"| total | {sum(cnt.values()) / steps:g} | {T:.3f} | |\n")
    traffic_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in reps:
        hdr, units, data = raw(rep)
        for row in data:
            name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else rep
            short = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "").replace("void ", "").split("(")[0]
            print(f"## `{short}` ({os.path.basename(rep)})\n")
            print("| metric | value |\n|---|---|")
            vals = {}
            for key, label in KEYS:
                if key in hdr:
                    i = hdr.index(key)
                    vals[key] = (row[i], units[i])
                    print(f"| {label} (`{key}`) | {row[i]} {units[i]} |")
            rd = to_bytes(*vals.get("dram__bytes_read.sum", ("0", "byte")))
            wr = to_bytes(*vals.get("dram__bytes_write.sum", ("0", "byte")))
            kname = ("near" if ("k_near" in name or "k_neval" in name) else "far_deferred" if "k_feval" in name
                     else "far" if "k_far" in name else name)
            traffic.setdefault(cfg, {})[f"{kname}_dram_bytes_per_launch"] = rd + wr
            traffic[cfg][f"{kname}_kernel"] = f"{short} ({tag} capture)"
            print()
    json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main()
