"""BASELINE configs[2]: 4M points on the unit sphere (nu = normal), theta 0.7, N0 2000, the
p in {2, 4, 6, 8, 10} error-vs-time curve.  Per order: device time of a full standalone
treecode call (median of 3), the order sweep's shared-pass times, and the error against the
direct sum on the reference harness's strided 1,000-target subset -- ours and the
reference's own (oracle/_ref treecode at the subset; the reference's direct sum).
Writes profiles/r02_cfg2_psweep.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_1811_12498_b200 as S
from oracle import oracle as O

N, THETA, N0 = 4_000_000, 0.7, 2000
threads = len(os.sched_getaffinity(0))
ps = S.generate("sphere", N, 12345, True)
d = dict(position=ps.position, force_weight=ps.force_weight, dipole_weight=ps.dipole_weight, normal=ps.normal)
idx = np.arange(1000, dtype=np.int64) * (N // 1000)
u_dir = S.contracted_direct_velocity_at(ps, S.KernelSelection.both(), idx)
u_dir_ref = O.ref_direct_at(d, idx, threads=threads)
rows = []
for p in (2, 4, 6, 8, 10):
    prm = S.TreecodeParams(order=p, theta=THETA, leaf_capacity=N0)
    ts = []
    for _ in range(3):
        r = S.treecode_velocity(ps, prm)
        ts.append(r.time_total_s)
    ctx = O.RefContext(d, p, THETA, N0, True, workers=threads)
    u_ref = ctx.eval(src_idx=idx, threads=threads)[0]
    ctx.close()
    e, e_ref = S.relative_error(u_dir, r.velocity[idx]), O.relative_error(u_dir_ref, u_ref)
    rows.append({"p": p, "device_time_s": float(np.median(ts)), "targets_per_s": N / float(np.median(ts)),
                 "far_s": r.time_far_s, "near_s": r.time_near_s, "moments_s": r.time_moments_s,
                 "E_vs_direct": e, "E_reference": e_ref, "E_rel_diff": abs(e - e_ref) / e_ref,
                 "rel_l2_vs_reference_subset": O.relative_error(u_ref, r.velocity[idx]),
                 "farfield_evals": r.stats.farfield_evals, "direct_pairs": r.stats.direct_pairs})
    print(rows[-1], flush=True)
u, far_s, rs = S.treecode_velocity_sweep(ps, S.TreecodeParams(order=10, theta=THETA, leaf_capacity=N0),
                                         [2, 4, 6, 8, 10])
sweep = {"orders": [2, 4, 6, 8, 10], "total_s": rs.time_total_s, "far_s_per_order": list(map(float, far_s)),
         "E_vs_direct": [S.relative_error(u_dir, u[k][idx]) for k in range(5)],
         "note": "st_treecode_velocity_sweep: one tree, one moment pass at p=10, one near field, a fold + "
                 "far field per order; each order bit-identical to its standalone call"}
json.dump({"config": "BASELINE configs[2]: N=4,000,000 on the unit sphere, nu = outward normal, theta 0.7, "
                     "N0 2000, both kernels, seed 12345", "subset": "1000 strided targets (bench.hpp:235-241)",
           "reference_cores": threads, "per_order": rows, "sweep": sweep},
          open(os.path.join(ROOT, "profiles", "r02_cfg2_psweep.json"), "w"), indent=1)
