"""One process per GPU: the exchange step of the split moment pass over torch.distributed.

`treecode_velocity_device_split` (st_treecode_velocity_device_split) calls the exchange
once per call, after this rank's weight rows and subtree-root moments are queued on the
call's stream.  `collective_exchange` moves every rank's rows into every rank's buffers with
one broadcast per rank and buffer, issued on that stream (NCCL over NVLink on the
driver's runs; gloo works for CPU-side plumbing checks).  Every rank computes the same cut
points, so no sizes are exchanged."""


class _DeviceView:
    """A raw device pointer as a 2-D float64 array (__cuda_array_interface__, zero copy)."""

    def __init__(self, ptr, rows, cols):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(rows), int(cols)),
                                         "typestr": "<f8", "strides": None, "version": 2}


def call_stream(ex, device):
    """The library call's stream as a torch stream (NULL = the legacy default stream)."""
    import torch
    if ex.stream:
        return torch.cuda.ExternalStream(ex.stream, device=device)
    return torch.cuda.default_stream(device)


def collective_exchange(dist, device):
    """Exchange callback for `treecode_velocity_device_split` over `dist` (torch.distributed)."""
    import torch

    def exchange(ex):
        wc, mc = ex.cuts("w"), ex.cuts("m")
        with torch.cuda.device(device), torch.cuda.stream(call_stream(ex, device)):
            w = torch.as_tensor(_DeviceView(ex.w, ex.ncl, ex.w_row), device=device)
            m = torch.as_tensor(_DeviceView(ex.m, max(1, ex.n_units), ex.m_row), device=device)
            for r in range(ex.n_shards):
                if wc[r + 1] > wc[r]:
                    dist.broadcast(w[wc[r]:wc[r + 1]], src=r)
                if mc[r + 1] > mc[r]:
                    dist.broadcast(m[mc[r]:mc[r + 1]], src=r)

    return exchange
