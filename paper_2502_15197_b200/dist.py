"""Request-sharded multi-GPU selection (one process per GPU, torch.distributed over NCCL / NVLink).

Rank g owns requests [g*B_local, (g+1)*B_local).  Verification and compaction are purely local; the only exchange
is the one the global capacity budget needs: an all-gather of every shard's candidate scores (conf rows f64 and
lengths, B_local*(8k+4) bytes per rank — 2 MB for B=16384, k=16), after which each rank runs the identical
single-device selection kernel over the gathered [B, k] matrix and keeps its own slice of windows.  Because every
rank evaluates the same kernel on bit-identical inputs, the windows equal the single-GPU (and CPU-reference)
selection for any world size by construction; global row ids are the gathered row order, so the reference's
(cum desc, row asc, depth asc) tie-break is preserved across shards.

On an NCCL group the exchange and the step are one native call on the torch communicator (`nccl_comm`;
csrc/dist.cu tetris_dist_*, which non-Python hosts call the same way); gloo groups (CPU tests) gather here.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


@dataclass
class ShardSelection:
    windows: torch.Tensor       # [B_local] i32 (view into the global result)
    win_offsets: torch.Tensor   # [B_local+1] i32, local exclusive scan
    global_windows: torch.Tensor
    row0: int                   # first global row of this shard
    status: Optional[torch.Tensor] = None


def gather_scores(conf_all: torch.Tensor, len_all: torch.Tensor, conf: torch.Tensor, lengths: torch.Tensor,
                  group=None) -> None:
    """All-gather every shard's scores and drafted depths into the [W*B, k] / [W*B] buffers.  NCCL: the two
    all-gathers go out as ONE coalesced NCCL group (one launch, one latency), the selection's only exchange per step;
    gloo (CPU / single-device tests): the list form."""
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        try:
            from torch.distributed.distributed_c10d import _coalescing_manager
        except ImportError:  # older torch: two collectives
            _coalescing_manager = None
        if _coalescing_manager is not None:
            with _coalescing_manager(group=group, device=conf.device):
                dist.all_gather_into_tensor(conf_all, conf.contiguous(), group=group)
                dist.all_gather_into_tensor(len_all, lengths.contiguous(), group=group)
        else:
            dist.all_gather_into_tensor(conf_all, conf.contiguous(), group=group)
            dist.all_gather_into_tensor(len_all, lengths.contiguous(), group=group)
    else:
        dist.all_gather(list(conf_all.chunk(world)), conf.contiguous(), group=group)
        dist.all_gather(list(len_all.chunk(world)), lengths.contiguous(), group=group)


def nccl_comm(group, device) -> Optional[int]:
    """The group's ncclComm_t (as an int) for `device`, for the native sharded entry points (tetris_dist_*, which
    issue their all-gathers on that communicator); None for non-NCCL backends.  A lazily initialised communicator is
    created by one small all-reduce first (every rank constructs its step at the same point, so this is collective)."""
    if group is None or dist.get_backend(group) != "nccl":
        return None
    dev = torch.device(device)
    backend = group._get_backend(dev)

    def ptr():
        try:
            with torch.cuda.device(dev):  # the communicator of this device
                return int(backend._comm_ptr())
        except RuntimeError:
            return 0

    p = ptr()
    if not p:
        dist.all_reduce(torch.zeros(1, device=dev), group=group)
        torch.cuda.synchronize(dev)
        p = ptr()
    if not p:
        raise RuntimeError("ProcessGroupNCCL exposes no communicator for the native sharded step")
    return p


def _all_gather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    else:  # gloo (CPU tests): list form
        dist.all_gather(list(out.chunk(world)), t.contiguous(), group=group)
    return out


def dist_select(conf_local: torch.Tensor, capacity: int, lengths_local: Optional[torch.Tensor] = None, *,
                group=None, select_fn: Optional[Callable] = None) -> ShardSelection:
    """Global TETRIS selection over all shards with a global capacity `capacity`.

    `select_fn(conf, capacity, lengths) -> (windows [B] i32 tensor, status or None)` defaults to the CUDA kernel;
    the gloo tests inject the CPU oracle to check the exchange logic without a GPU."""
    B_local, k = conf_local.shape
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if lengths_local is None:
        lengths_local = torch.full((B_local,), k, dtype=torch.int32, device=conf_local.device)
    conf_all = torch.empty((world * B_local, k), dtype=conf_local.dtype, device=conf_local.device)
    len_all = torch.empty((world * B_local,), dtype=torch.int32, device=conf_local.device)
    comm = nccl_comm(group, conf_local.device) if select_fn is None else None
    if comm is not None:
        # native: the exchange + the global selection in one library call on the current stream (csrc/dist.cu)
        from . import _native as N
        from .ops import Workspace, new_status

        dev = conf_local.device
        windows = torch.empty(world * B_local, dtype=torch.int32, device=dev)
        status = new_status(dev)
        ws = Workspace(dev, N.OP_SELECT, world * B_local, k, 0)
        N.call("tetris_dist_select_f64", conf_local.contiguous().data_ptr(),
               lengths_local.to(torch.int32).contiguous().data_ptr(), B_local, k, int(capacity), 0, comm,
               conf_all.data_ptr(), len_all.data_ptr(), windows.data_ptr(), None, None, status.data_ptr(), ws.ptr,
               ws.nbytes, torch.cuda.current_stream(dev).cuda_stream)
    else:
        gather_scores(conf_all, len_all, conf_local, lengths_local.to(torch.int32), group)
        if select_fn is None:
            from . import ops

            res = ops.select(conf_all, capacity, len_all)
            windows, status = res.windows, res.status
        else:
            windows, status = select_fn(conf_all, capacity, len_all)
    r0 = rank * B_local
    local = windows[r0:r0 + B_local]
    offs = torch.zeros(B_local + 1, dtype=torch.int32, device=local.device)
    offs[1:] = torch.cumsum(local, 0, dtype=torch.int32)
    return ShardSelection(local, offs, windows, r0, status)
