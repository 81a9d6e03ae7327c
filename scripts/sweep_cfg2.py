"""BASELINE configs[2]: error-vs-time curve over p in {2,4,6,8,10}, N = 4M sphere surface,
theta 0.7, N0 2000.  One tree / moment pass / near pass (st_treecode_velocity_sweep);
E vs the O(N^2) direct sum on a strided 1,000-target sample (the reference's own
--direct-sample idiom, bench.hpp:235-244), and the reference treecode's E on the same
sample (oracle/_ref) when present.  Writes one JSON document to stdout."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1811_12498_b200 as S
from bench import CONFIGS, make_inputs

cfg = dict(CONFIGS["cfg2"])
if len(sys.argv) > 1:
    cfg["n"] = int(sys.argv[1])
orders = [2, 4, 6, 8, 10]
ps, _ = make_inputs(cfg)
n = cfg["n"]
prm = S.TreecodeParams(order=10, theta=cfg["theta"], leaf_capacity=cfg["n0"])
sample = np.arange(0, n, max(1, n // 1000))[:1000]
S.treecode_velocity_sweep(ps, prm, orders)  # warm-up (first launches load the kernels)
t = time.time()
u, far_s, res = S.treecode_velocity_sweep(ps, prm, orders)
wall = time.time() - t
direct = S.contracted_direct_velocity_at(ps, S.KernelSelection.both(), sample)
out = {"config": cfg["desc"], "n": n, "sample_targets": len(sample), "sweep_wall_s": wall,
       "shared_s": {"build": res.time_build_s, "moments_at_p10": res.time_moments_s,
                    "traverse_incl_near_and_all_far": res.time_traverse_s},
       "stats": res.stats.__dict__, "orders": []}
singles = {}
for i, p in enumerate(orders):
    r = S.treecode_velocity(ps, S.TreecodeParams(order=p, theta=cfg["theta"], leaf_capacity=cfg["n0"]))
    singles[p] = r.time_total_s
    e = S.relative_error(direct, u[i][sample])
    out["orders"].append({"p": p, "E_vs_direct": e, "far_kernel_s": float(far_s[i]),
                          "standalone_treecode_s": r.time_total_s,
                          "standalone_targets_per_s": n / r.time_total_s,
                          "bit_identical_to_standalone": bool(np.array_equal(r.velocity, u[i]))})
try:
    from oracle import oracle as O
    if O.have_ref():
        d = dict(position=ps.position, force_weight=ps.force_weight, dipole_weight=ps.dipole_weight,
                 normal=ps.normal)
        for row in out["orders"]:
            ctx = O.RefContext(d, row["p"], cfg["theta"], cfg["n0"], True, workers=os.cpu_count())
            ur, _, _ = ctx.eval(src_idx=sample, threads=os.cpu_count())
            ctx.close()
            row["E_reference_vs_direct"] = S.relative_error(direct, ur)
            row["E_rel_diff_vs_reference"] = abs(row["E_vs_direct"] - row["E_reference_vs_direct"]) / row[
                "E_reference_vs_direct"]
            row["rel_L2_vs_reference_on_sample"] = S.relative_error(ur, u[orders.index(row["p"])][sample])
except Exception as ex:  # reported, not fatal
    out["reference_error"] = str(ex)
print(json.dumps(out, indent=1))
