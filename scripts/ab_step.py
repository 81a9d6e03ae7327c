"""A/B probe: median device-timed treecode step and its far/near kernel times for one
configuration with whatever library ST_LIB_PATH names (scripts/ab_far_r02.sh).
python scripts/ab_step.py cfg4 [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1811_12498_b200 as S
from bench import CONFIGS, make_inputs

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS[name]
ps, tg = make_inputs(cfg)
n = cfg["n"]
nt = cfg["targets"] or n
dsrc = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
dtg = torch.from_numpy(tg).cuda() if tg is not None else None
dout = torch.zeros((nt, 3), dtype=torch.float64, device="cuda")
prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"])
b, st = dsrc.data_ptr(), n * 24
stream = torch.cuda.current_stream().cuda_stream
rows = []
for k in range(reps + 2):
    r = S.treecode_velocity_device(b, b + st, b + 2 * st, b + 3 * st, n, prm, dout.data_ptr(),
                                   targets_ptr=None if dtg is None else dtg.data_ptr(),
                                   n_targets=nt if dtg is not None else 0, stream=stream)
    torch.cuda.synchronize()
    if k >= 2:
        rows.append((r.time_total_s, r.time_far_s, r.time_near_s))
a = np.median(np.array(rows), axis=0) * 1e3
print(json.dumps({"config": name, "lib": os.path.basename(os.environ.get("ST_LIB_PATH", "default")),
                  "total_ms": round(a[0], 3), "far_ms": round(a[1], 3), "near_ms": round(a[2], 3),
                  "checksum": float(np.abs(dout.cpu().numpy()).sum())}), flush=True)
