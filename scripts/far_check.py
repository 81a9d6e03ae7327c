"""Bitwise check + timing of a far-field kernel variant against another (scratch probe).

python scripts/far_check.py out.npz   (run once per variant, e.g. with ST_FAR_OLD=1)
python scripts/far_check.py --compare a.npz b.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402

CASES = [  # kind, n, seed, order, theta, n0, kernels, disjoint targets
    ("cube", 1000000, 12345, 8, 0.5, 2000, "both", 0),
    ("sphere", 400000, 5, 10, 0.7, 2000, "both", 0),
    ("mixture", 300000, 7, 8, 0.6, 2000, "both", 300000),
    ("cube", 100000, 9, 1, 0.5, 300, "both", 0),
    ("cube", 50000, 10, 16, 0.4, 500, "both", 0),
    ("cube", 100000, 11, 6, 0.5, 64, "sto", 0),
    ("unit", 30000, 12, 0, 0.9, 1, "str", 0),
]

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    ok = True
    for k in a.files:
        if k.startswith("u"):
            same = np.array_equal(a[k], b[k])
            ok &= same
            rel = np.linalg.norm(a[k] - b[k]) / np.linalg.norm(a[k])
            print(k, "bit-identical" if same else f"DIFFER max {np.max(np.abs(a[k] - b[k])):.3e} rel L2 {rel:.2e}",
                  f"far {a['f' + k[1:]][0] * 1e3:.2f} -> {b['f' + k[1:]][0] * 1e3:.2f} ms")
    sys.exit(0 if ok else 1)

out = {}
for i, (kind, n, seed, p, th, n0, ker, nt) in enumerate(CASES):
    ps = S.generate(kind, n, seed, ker != "sto")
    sel = {"both": S.KernelSelection.both(), "sto": S.KernelSelection.stokeslet_only(),
           "str": S.KernelSelection.stresslet_only()}[ker]
    prm = S.TreecodeParams(order=p, theta=th, leaf_capacity=n0, kernels=sel)
    tg = S.generate("points", nt, seed + 1).position if nt else None
    for rep in range(2):
        r = S.treecode_velocity_targets(ps, tg, prm) if nt else S.treecode_velocity(ps, prm)
    out[f"u{i}"] = r.velocity
    out[f"f{i}"] = np.array([r.time_far_s])
    print(i, kind, n, p, f"far {r.time_far_s * 1e3:.2f} ms total {r.time_total_s * 1e3:.2f} ms", flush=True)
np.savez(sys.argv[1], **out)
