"""CPU, world_size 2 over gloo: the N > 1 plumbing of bench.py / DESIGN.md "Multi-GPU".

Every rank derives the same work-balanced cut of the key-ordered 32-target
batches (no communication), owns a disjoint shard, and the batch-order slices
are all-gathered (bench.allgather_batch_slices) and scattered to original order, so
the combined result is bit-identical to the single-rank result.  The batch order and the
cut use the CUDA path's own recipe (tests/shard_model.py: octree keys, k_count's cost
model, st_shard_cuts), pinned to the library by a GPU test; the per-target velocities
here come from the oracle (no GPU in this container)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1811_12498_b200 as S
    import shard_model as M
    from oracle import oracle as O
    n, order_p, theta, n0 = 3000, 4, 0.5, 200
    ps = S.generate("cube", n, 12345, True)
    d = dict(position=ps.position, force_weight=ps.force_weight, dipole_weight=ps.dipole_weight,
             normal=ps.normal)
    # replicated sources: rank 0's copy broadcast to everyone
    src = torch.from_numpy(ps.position.copy()) if rank == 0 else torch.zeros((n, 3), dtype=torch.float64)
    dist.broadcast(src, 0)
    assert np.array_equal(src.numpy(), ps.position)
    # the CUDA path's batch order (octree keys in the root cube of the targets' tight box) and its per-warp
    # cost model (k_count over the exact interaction lists), restated on the host and checked
    # against the library by tests/test_gpu_parity.py::test_shard_plan_matches_host_model
    order = M.key_batch_order(ps.position)
    T = O.or_build_tree(d, n0, True)
    to_tree = np.empty(n, np.uint32)
    to_tree[T.to_original] = np.arange(n, dtype=np.uint32)
    far, near = O.or_lists(d, n0, True, theta, tree_idx=to_tree, cap=4096)
    cost = M.warp_costs(order, far, near, T.end - T.begin, order_p + 2)
    nwarps = len(cost)
    cuts = S.shard_cuts(cost, world)  # st_shard_cuts, identical on every rank
    u_all, _, _ = O.or_treecode(d, order_p, theta, n0, per_target=True, threads=2)
    # this rank's slice in batch order, gathered exactly as bench.py does it
    from bench import allgather_batch_slices
    t0, t1 = min(n, 32 * int(cuts[rank])), min(n, 32 * int(cuts[rank + 1]))
    ubatch = torch.zeros((n, 3), dtype=torch.float64)
    ubatch[t0:t1] = torch.from_numpy(u_all[order[t0:t1]])
    ranges = allgather_batch_slices(dist, ubatch, t0, t1, world)
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    out = torch.zeros((n, 3), dtype=torch.float64)
    out[torch.from_numpy(order)] = ubatch  # the unbatch scatter (st_unbatch_device on a GPU)
    allcuts = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allcuts, torch.from_numpy(cuts))
    if rank == 0:
        q.put((out.numpy().tobytes() == u_all.tobytes(),
               all(torch.equal(allcuts[0], c) for c in allcuts), cuts.tolist(), nwarps))
    dist.destroy_process_group()


def test_two_rank_shards_combine_bit_exactly():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    same, cuts_agree, cuts, nwarps = res
    assert cuts_agree
    assert cuts[0] == 0 and cuts[-1] == nwarps and 0 < cuts[1] < nwarps
    assert same
