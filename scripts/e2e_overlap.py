"""e2e step with and without the weight upload overlapping the tree build (scratch probe)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402
from bench import CONFIGS, make_inputs  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]
ps, tg = make_inputs(cfg)
n = cfg["n"]
host = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).pin_memory()
dsrc = torch.empty(host.shape, dtype=torch.float64, device="cuda")
dout = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
hout = torch.empty((n, 3), dtype=torch.float64).pin_memory()
prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"])
main = torch.cuda.current_stream()
side = torch.cuda.Stream()
b, st = dsrc.data_ptr(), n * 24
ptrs = (b, b + st, b + 2 * st, b + 3 * st)


def step(overlap):
    if overlap:
        ws, wr = torch.cuda.Event(), torch.cuda.Event()
        ws.record(main)
        side.wait_event(ws)
        dsrc[:n].copy_(host[:n], non_blocking=True)
        with torch.cuda.stream(side):
            dsrc[n:].copy_(host[n:], non_blocking=True)
            wr.record(side)
        S.treecode_velocity_device(*ptrs, n, prm, dout.data_ptr(), stream=main.cuda_stream, weights_event=wr.cuda_event)
    else:
        dsrc.copy_(host, non_blocking=True)
        S.treecode_velocity_device(*ptrs, n, prm, dout.data_ptr(), stream=main.cuda_stream)
    hout.copy_(dout, non_blocking=True)


for overlap in (False, True, False, True):
    for _ in range(2):
        step(overlap)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        step(overlap)
        z.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(z))
    h2d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h2d[0].record(main)
    dsrc.copy_(host, non_blocking=True)
    h2d[1].record(main)
    torch.cuda.synchronize()
    print("overlap" if overlap else "serial ", "e2e ms", [round(t, 2) for t in ts], "H2D alone", round(h2d[0].elapsed_time(h2d[1]), 2))
