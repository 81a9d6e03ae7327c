"""Where the reference-facing host call spends its time (scratch probe): cfg1 through
st_treecode_velocity_ex from pinned and from pageable host arrays."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402
from bench import CONFIGS, make_inputs  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]
ps, tg = make_inputs(cfg)
prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"])
n = cfg["n"]
pin = torch.empty((4 * n, 3), dtype=torch.float64).pin_memory().numpy()
pin[:] = np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])
pps = S.ParticleSet(pin[:n], pin[n:2 * n], pin[2 * n:3 * n], pin[3 * n:])
for name, p in (("pageable", ps), ("pinned", pps)):
    for k in range(4):
        t0 = time.perf_counter()
        r = S.treecode_velocity(p, prm)
        w = time.perf_counter() - t0
        if k:
            print(f"{name}: wall {w*1e3:.2f} ms  device total {r.time_total_s*1e3:.2f}  h2d {r.time_h2d_s*1e3:.2f}  "
                  f"d2h {r.time_d2h_s*1e3:.2f}  build {r.time_build_s*1e3:.2f}", flush=True)
