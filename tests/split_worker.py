"""Worker for tests/test_gpu_parity.py::test_split_moment_pass_ranks (under
torch.distributed.run, gloo, ranks sharing one GPU): every rank computes its share of the
moment pass (st_treecode_velocity_device_split), the ranks exchange weight rows and
subtree-root moments with paper_1811_12498_b200.distributed.collective_exchange, and each
rank's epilogue stores its target shard into rank 0's buffer (CUDA IPC).  Rank 0 checks the
result bit for bit against one GPU.  The ranks never wait on each other's kernels: the
exchange is a host-driven collective between the calls' phases."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402
from paper_1811_12498_b200.distributed import collective_exchange  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    kind, n, order, theta, n0 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
    ps = S.generate(kind, n, 11, True)
    tg = S.generate("points", n // 2, 67890).position if kind == "mixture" else None
    nt = n if tg is None else len(tg)
    dsrc = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
    dtg = torch.from_numpy(tg).cuda() if tg is not None else None
    prm = S.TreecodeParams(order=order, theta=theta, leaf_capacity=n0)
    dout = torch.full((nt, 3), float("nan"), dtype=torch.float64, device="cuda")
    obj = [S.ipc_export(dout.data_ptr()) if rank == 0 else None]
    dist.broadcast_object_list(obj, 0)
    out = dout.data_ptr() if rank == 0 else S.ipc_open(*obj[0])
    b, st = dsrc.data_ptr(), n * 24
    for _ in range(2):  # twice: buffers and cut points are per call
        S.treecode_velocity_device_split(b, b + st, b + 2 * st, b + 3 * st, n, prm, out, collective_exchange(dist, dev),
                                         targets_ptr=None if dtg is None else dtg.data_ptr(),
                                         n_targets=0 if dtg is None else nt, shard=rank, n_shards=world,
                                         stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        dist.barrier()
    if rank == 0:
        ref = S.treecode_velocity_targets(ps, tg, prm).velocity
        got = dout.cpu().numpy()
        assert np.array_equal(got, ref), f"split moment pass differs: {np.nanmax(np.abs(got - ref))}"
        print("SPLIT_OK", flush=True)
    dist.barrier()
    if rank != 0:
        S.ipc_close(out)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
