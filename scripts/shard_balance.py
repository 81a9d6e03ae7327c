"""Load balance of the multi-GPU shard cuts, measured on one GPU: every shard of an
n-way split run in turn; prints each shard's far + near kernel time (scratch probe).
python scripts/shard_balance.py cfg1 8"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402
from bench import CONFIGS, make_inputs  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
k = int(sys.argv[2])
ps, tg = make_inputs(cfg)
n = cfg["n"]
nt = cfg["targets"] or n
dsrc = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
dtg = torch.from_numpy(tg).cuda() if tg is not None else None
dout = torch.zeros((nt, 3), dtype=torch.float64, device="cuda")
prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"])
b, st = dsrc.data_ptr(), n * 24
stream = torch.cuda.current_stream().cuda_stream
for rep in range(2):
    times, calls = [], []
    for r in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = S.treecode_velocity_device(b, b + st, b + 2 * st, b + 3 * st, n, prm, dout.data_ptr(),
                                         targets_ptr=None if dtg is None else dtg.data_ptr(),
                                         n_targets=nt if dtg is not None else 0, shard=r, n_shards=k, stream=stream)
        e1.record()
        torch.cuda.synchronize()
        times.append(1e3 * (res.time_far_s + res.time_near_s))
        calls.append(e0.elapsed_time(e1))  # the whole shard call: what one rank's step costs
full = S.treecode_velocity_device(b, b + st, b + 2 * st, b + 3 * st, n, prm, dout.data_ptr(),
                                  targets_ptr=None if dtg is None else dtg.data_ptr(),
                                  n_targets=nt if dtg is not None else 0, stream=stream)
ideal = 1e3 * (full.time_far_s + full.time_near_s) / k
print(sys.argv[1], k, "shards far+near ms:", [round(x, 2) for x in times], "max/ideal",
      round(max(times) / ideal, 3), "total/k", round(sum(times) / k, 2), "ideal", round(ideal, 2))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
S.treecode_velocity_device(b, b + st, b + 2 * st, b + 3 * st, n, prm, dout.data_ptr(),
                           targets_ptr=None if dtg is None else dtg.data_ptr(),
                           n_targets=nt if dtg is not None else 0, stream=stream)
e1.record()
torch.cuda.synchronize()
one = e0.elapsed_time(e1)
print(sys.argv[1], k, "whole shard calls ms:", [round(x, 2) for x in calls], "one GPU", round(one, 2),
      "-> projected step", round(max(calls), 2), "efficiency", round(one / (k * max(calls)), 3),
      "(no NVLink stores / all-reduce; shards run one at a time)")
