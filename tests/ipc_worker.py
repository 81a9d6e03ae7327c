"""Worker for tests/test_gpu_parity.py::test_ipc_fused_gather (run under torch.distributed.run).

Rank 0 exports its output buffer over CUDA IPC; every rank evaluates its shard with
st_treecode_velocity_device and the epilogue kernel stores straight into rank 0's
buffer (the fused gather bench.py uses over NVLink).  Both ranks may share one GPU:
their kernels never wait on each other -- they only store, then meet at a CPU barrier."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(rank % torch.cuda.device_count())
    ps = S.generate("cube", 20000, 11, True)
    n = ps.size()
    dsrc = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
    prm = S.TreecodeParams(order=5, theta=0.5, leaf_capacity=400)
    dout = torch.full((n, 3), float("nan"), dtype=torch.float64, device="cuda")
    obj = [S.ipc_export(dout.data_ptr()) if rank == 0 else None]
    dist.broadcast_object_list(obj, 0)
    out = dout.data_ptr() if rank == 0 else S.ipc_open(*obj[0])
    b, st = dsrc.data_ptr(), n * 24
    S.treecode_velocity_device(b, b + st, b + 2 * st, b + 3 * st, n, prm, out, shard=rank, n_shards=world,
                               stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        ref = S.treecode_velocity(ps, prm).velocity
        got = dout.cpu().numpy()
        assert np.array_equal(got, ref), f"fused gather differs: {np.nanmax(np.abs(got - ref))}"
        print("IPC_OK", flush=True)
    dist.barrier()
    if rank != 0:
        S.ipc_close(out)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
