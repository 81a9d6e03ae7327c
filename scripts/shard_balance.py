"""Projected N-GPU step, measured on one GPU: every shard of an n-way split runs in turn, each
as the whole call one rank makes (CUDA events around it); the projected step is the slowest
shard (each shard's median of three timed passes).  python scripts/shard_balance.py cfg4 8 [split|replicated]

split (default): the moment pass is split over the ranks (st_treecode_velocity_device_split).
A first pass runs every shard and captures the weight rows and subtree-root moments it
produced; the timed pass then runs every shard again with an exchange callback that copies
the other ranks' captured rows into its buffers on the call's stream (a device copy standing
in for the NCCL broadcasts over NVLink, whose cost is added from the bytes at 700 GB/s).
The velocities of the timed pass, assembled from all shards, must equal one GPU bit for bit.
replicated: every shard also computes the whole moment pass (round 1)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402
from bench import CONFIGS, make_inputs  # noqa: E402
from paper_1811_12498_b200.distributed import _DeviceView, call_stream  # noqa: E402

NVLINK_GBS = 700.0  # measured peer copy per direction (B200_PROFILING.md: ~725-770 GB/s)

name = sys.argv[1]
k = int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "split"
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


def views(ex):
    w = torch.as_tensor(_DeviceView(ex.w, ex.ncl, ex.w_row), device="cuda")
    m = torch.as_tensor(_DeviceView(ex.m, max(1, ex.n_units), ex.m_row), device="cuda")
    return w, m, ex.cuts("w"), ex.cuts("m")


store = {}
xbytes = {}


def capture(ex):
    w, m, wc, mc = views(ex)
    r = ex.shard
    with torch.cuda.stream(call_stream(ex, torch.cuda.current_device())):
        store[r] = (w[wc[r]:wc[r + 1]].clone(), m[mc[r]:mc[r + 1]].clone())
    # bytes this rank receives in the real exchange
    xbytes[r] = 8 * ((ex.ncl - (wc[r + 1] - wc[r])) * ex.w_row + (ex.n_units - (mc[r + 1] - mc[r])) * ex.m_row)


def replay(ex):
    w, m, wc, mc = views(ex)
    with torch.cuda.stream(call_stream(ex, torch.cuda.current_device())):
        for q in range(ex.n_shards):
            if q != ex.shard:
                w[wc[q]:wc[q + 1]].copy_(store[q][0])
                m[mc[q]:mc[q + 1]].copy_(store[q][1])


full_out = torch.zeros((nt, 3), dtype=torch.float64, device="cuda")
full = S.treecode_velocity_device(*ptrs, n, prm, full_out.data_ptr(), stream=stream, **tkw)
one_ms = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.treecode_velocity_device(*ptrs, n, prm, full_out.data_ptr(), stream=stream, **tkw)
    e1.record()
    torch.cuda.synchronize()
    one_ms.append(e0.elapsed_time(e1))
one = float(np.median(one_ms))

dout = torch.zeros((nt, 3), dtype=torch.float64, device="cuda")


def shard_call(r, fn):
    if mode == "split":
        return S.treecode_velocity_device_split(*ptrs, n, prm, dout.data_ptr(), fn, shard=r, n_shards=k, stream=stream,
                                                **tkw)
    return S.treecode_velocity_device(*ptrs, n, prm, dout.data_ptr(), shard=r, n_shards=k, stream=stream, **tkw)


if mode == "split":
    for r in range(k):
        shard_call(r, capture)
    torch.cuda.synchronize()
# three timed passes; each shard's median call (a host-side hiccup in one call -- e.g. the
# pool mapping memory -- would otherwise decide the projected step)
reps = [[], [], []]
kern = []
for rep in range(3):
    kern = []
    dout.zero_()
    for r in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = shard_call(r, replay)
        e1.record()
        torch.cuda.synchronize()
        reps[rep].append(e0.elapsed_time(e1))
        kern.append(1e3 * (res.time_far_s + res.time_near_s))
    if rep == 0:
        identical = bool(torch.equal(dout, full_out))
calls = [float(np.median([reps[q][r] for q in range(3)])) for r in range(k)]
nv = [1e3 * xbytes.get(r, 0) / (NVLINK_GBS * 1e9) for r in range(k)]
proj = max(c + x for c, x in zip(calls, nv))
line = {"config": name, "shards": k, "moments": mode, "one_gpu_ms": round(one, 3),
        "shard_call_ms": [round(c, 3) for c in calls], "shard_call_ms_max": [round(max(q[r] for q in reps), 3) for r in range(k)], "exchange_ms_modelled": [round(x, 3) for x in nv],
        "far_near_kernel_ms": [round(x, 3) for x in kern],
        "projected_step_ms": round(proj, 3), "efficiency": round(one / (k * proj), 3),
        "bit_identical_to_one_gpu": identical,
        "note": "shards run one at a time on one GPU; exchange = device copy + modelled NVLink time"}
print(json.dumps(line), flush=True)
