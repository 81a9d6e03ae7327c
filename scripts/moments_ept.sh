# k_moments kernel time per entries-per-thread choice (ncu launch list, one step each)
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg4; do for e in ${EPTS:-4 2 1}; do
  ST_LIB_PATH=${LIB:+$PWD/scratch_libs/$LIB.so} ST_MOMENTS_EPT=$e ncu --metrics gpu__time_duration.sum,launch__registers_per_thread --clock-control none --csv -k regex:k_moments --log-file gpurun_out/mom_${c}_$e.csv python scripts/profile_step.py $c 1 > /dev/null 2>&1
  python - "$c" "$e" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/mom_{sys.argv[1]}_{sys.argv[2]}.csv")))
h = next(r for r in rows if "Kernel Name" in r)
t = [float(r[h.index("Metric Value")].replace(",", "")) for r in rows[rows.index(h) + 1:] if len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum"]
g = [r[h.index("Metric Value")] for r in rows[rows.index(h) + 1:] if len(r) == len(h) and r[h.index("Metric Name")] == "launch__registers_per_thread"]
import os; print(os.environ.get("LIB", "tree"), sys.argv[1], "EPT", sys.argv[2], "k_moments ms", round(sum(t) / 1e6, 3), "regs", g[:1])
PY
done; done
