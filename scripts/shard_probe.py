"""One shard of an n-way split (replicated moments) at a BASELINE config, timed by the
library's phase events; for launch lists of a single rank's call under ncu.
python scripts/shard_probe.py cfg4 8 3 [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402
from bench import CONFIGS, make_inputs  # noqa: E402

name, k, r = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
cfg = CONFIGS[name]
ps, tg = make_inputs(cfg)
n = cfg["n"]
nt = cfg["targets"] or n
dsrc = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
dtg = torch.from_numpy(tg).cuda() if tg is not None else None
prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"])
b, st = dsrc.data_ptr(), n * 24
ptrs = (b, b + st, b + 2 * st, b + 3 * st)
stream = torch.cuda.current_stream().cuda_stream
tkw = dict(targets_ptr=None if dtg is None else dtg.data_ptr(), n_targets=nt if dtg is not None else 0)
out = torch.zeros((nt, 3), dtype=torch.float64, device="cuda")
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = S.treecode_velocity_device(*ptrs, n, prm, out.data_ptr(), shard=r, n_shards=k, stream=stream, **tkw)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} shard {r}/{k}: {e0.elapsed_time(e1):.3f} ms build {1e3 * res.time_build_s:.3f} "
          f"far {1e3 * res.time_far_s:.3f} near {1e3 * res.time_near_s:.3f}", flush=True)
