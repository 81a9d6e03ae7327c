"""NCCL inside the library (st_treecode_velocity_nccl): the communicator, the split moment
pass's exchange by NCCL broadcasts and the gather by one NCCL sum.  On a one-GPU box the
collective runs with one rank (NCCL refuses two ranks on one GPU); with two GPUs visible,
two processes run it for real."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(S, kind, n, disjoint):
    ps = S.generate(kind, n, 31, True)
    src = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
    tg = torch.from_numpy(S.generate("points", 9000, 7).position).cuda() if disjoint else None
    b, st = src.data_ptr(), n * 24
    return (b, b + st, b + 2 * st, b + 3 * st), src, tg


@pytest.mark.parametrize("kind,n,disjoint", [("cube", 40000, False), ("mixture", 30000, True)])
def test_nccl_one_rank_bit_identical(S, kind, n, disjoint):
    ptrs, src, tg = _inputs(S, kind, n, disjoint)
    nt = len(tg) if tg is not None else n
    prm = S.TreecodeParams(order=6, theta=0.6, leaf_capacity=300)
    tkw = dict(targets_ptr=None if tg is None else tg.data_ptr(), n_targets=0 if tg is None else nt)
    stream = torch.cuda.current_stream().cuda_stream
    one = torch.zeros((nt, 3), dtype=torch.float64, device="cuda")
    r1 = S.treecode_velocity_device(*ptrs, n, prm, one.data_ptr(), stream=stream, **tkw)
    comm = S.NcclComm(S.nccl_unique_id(), 1, 0)
    out = torch.full((nt, 3), 7.0, dtype=torch.float64, device="cuda")
    r2 = S.treecode_velocity_nccl(*ptrs, n, prm, out.data_ptr(), comm, stream=stream, **tkw)
    torch.cuda.synchronize()
    comm.close()
    assert torch.equal(out, one)
    assert r2.stats == r1.stats


_WORKER = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1811_12498_b200 as S
rank, world, idfile, outfile = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
torch.cuda.set_device(rank)
import time, os
if rank == 0:
    open(idfile + ".tmp", "wb").write(S.nccl_unique_id()); os.replace(idfile + ".tmp", idfile)
while not os.path.exists(idfile):
    time.sleep(0.05)
uid = open(idfile, "rb").read()
n = 60000
ps = S.generate("cube", n, 31, True)
src = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
b, st = src.data_ptr(), n * 24
prm = S.TreecodeParams(order=6, theta=0.6, leaf_capacity=300)
comm = S.NcclComm(uid, world, rank)
out = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
r = S.treecode_velocity_nccl(b, b + st, b + 2 * st, b + 3 * st, n, prm, out.data_ptr(), comm,
                             stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
np.save(outfile, out.cpu().numpy())
comm.close()
"""


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="two ranks need two GPUs (NCCL: one rank per GPU)")
def test_nccl_two_ranks_bit_identical(S, tmp_path):
    idfile = str(tmp_path / "id")
    procs = [subprocess.Popen([sys.executable, "-c", _WORKER, ROOT, str(r), "2", idfile, str(tmp_path / f"u{r}.npy")])
             for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    n = 60000
    ptrs, src, _ = _inputs(S, "cube", n, False)
    one = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    S.treecode_velocity_device(*ptrs, n, S.TreecodeParams(order=6, theta=0.6, leaf_capacity=300), one.data_ptr(),
                               stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = one.cpu().numpy()
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"u{r}.npy"), ref)
