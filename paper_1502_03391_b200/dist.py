"""Multi-GPU plumbing for the sharded Guttman loop (one process per GPU).

Three exchanges: attach_nccl_native (the default: the C ABI's own NCCL
reduce-scatter of the products + all-gather of X per iteration, captured in
the solve's CUDA graph, csrc/capi_nccl.cu), attach_nccl (a Python all-reduce
hook over torch.distributed, below) and attach_peers (the products and
configuration rows move through peer memory inside the loop's own kernels,
csrc/jofc_peer.cuh).

Each rank owns a balanced contiguous range of the packed Delta block stream
(jofc_set_shard); every iteration the partial product P = B(X)X (m*n_pad*d
doubles) and the partial fidelity ride in one exchange buffer that must be
sum-all-reduced before the epilogue (W^-1 mix, stress, stop rule) runs
redundantly on every rank.  The buffer is a torch tensor handed to the C ABI
(jofc_set_exchange_buffer) so torch.distributed/NCCL reduces it in place on
the context's stream.
"""
from __future__ import annotations

import threading

from ._capi import check


class _CudaView:
    """__cuda_array_interface__ wrapper: raw device pointer -> torch tensor."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 2,
                                         "strides": None}


def cuda_view(ptr, count, device):
    import torch
    return torch.as_tensor(_CudaView(ptr, count), device=device)


def attach_nccl(dev, d, group=None):
    """Give `dev` (a paper_1502_03391_b200.Device with a shard set) a torch-owned
    exchange buffer and an all-reduce hook over torch.distributed."""
    import torch
    import torch.distributed as dist
    count = dev.lib.jofc_exchange_count(dev.h, d)
    buf = torch.zeros(count, dtype=torch.float64, device=f"cuda:{dev.device}")
    check(dev.lib.jofc_set_exchange_buffer(dev.h, buf.data_ptr(), count))
    stream = torch.cuda.ExternalStream(dev.stream, device=f"cuda:{dev.device}")

    def hook(ptr, cnt, strm):
        with torch.cuda.stream(stream):
            dist.all_reduce(buf[:cnt], group=group)
    dev.set_allreduce(hook)
    dev._xbuf = buf
    return buf


def attach_nccl_native(dev, group=None):
    """The C-native NCCL exchange (csrc/capi_nccl.cu): rank 0 makes an NCCL
    unique id, torch.distributed broadcasts it, every rank's context joins the
    communicator.  From then on each Guttman iteration's reduce-scatter of the
    products and all-gather of the new configuration rows are issued by the C
    ABI itself, on the context stream, inside the solve's CUDA graph -- no
    Python in the loop."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [dev.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    dev.nccl_init(obj[0], rank, world)
    dist.barrier(group=group)


def exchange_handles(handle, group=None):
    """All-gather of one bytes object per rank (rank order)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return out


def attach_peers(dev, group=None):
    """Peer-memory exchange instead of NCCL (jofc_peer_*): every rank exports
    its slab as a CUDA IPC handle, the handles are all-gathered, every rank
    maps the others' slabs.  The Guttman loop then exchanges products and
    configuration rows through NVLink loads/stores inside its own kernels."""
    import torch.distributed as dist
    handle, _ = dev.peer_export()
    handles = exchange_handles(handle, group)
    dev.peer_attach(dist.get_rank(group), len(handles), handles)
    dist.barrier(group=group)  # every slab zeroed before any rank's first flag
    return handles


class ThreadGroup:
    """Single-process stand-in for a W-rank group: W contexts, each driven by
    its own host thread, reduce their exchange buffers on the host side (the
    device never waits on another context's kernels).  Test use only."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.views = [None] * world

    def hook_for(self, rank, device):
        import torch

        def hook(ptr, count, stream):
            torch.cuda.ExternalStream(stream, device=device).synchronize()
            self.views[rank] = cuda_view(ptr, count, device)
            self.bar.wait()
            if rank == 0:
                total = self.views[0].clone()
                for v in self.views[1:]:
                    total += v
                for v in self.views:
                    v.copy_(total)
                torch.cuda.synchronize(device)
            self.bar.wait()
        return hook
