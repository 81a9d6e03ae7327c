"""One device-resident treecode step (for ncu captures): python scripts/profile_step.py [cfg]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1811_12498_b200 as S
from bench import CONFIGS, make_inputs
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ps, tg = make_inputs(cfg)
n = cfg["n"]; nt = cfg["targets"] or n
dsrc = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
dtg = torch.from_numpy(tg).cuda() if tg is not None else None
dout = torch.zeros((nt, 3), dtype=torch.float64, device="cuda")
prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"])
b = dsrc.data_ptr(); st = n * 24
for _ in range(reps):
    r = S.treecode_velocity_device(b, b + st, b + 2 * st, b + 3 * st, n, prm, dout.data_ptr(),
                                   targets_ptr=None if dtg is None else dtg.data_ptr(), n_targets=nt if dtg is not None else 0,
                                   stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", r.time_total_s, r.time_far_s, r.time_near_s, r.gpu_launches)
