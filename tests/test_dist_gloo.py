"""CPU, world_size 2 over gloo: the request-sharded selection exchange (paper_2502_15197_b200/dist.py).

Each rank owns half of the requests; the all-gather + global selection must give every rank exactly the windows
of a single-device selection over the whole batch (here the CPU oracle stands in for the CUDA kernel)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_select(conf, C, lengths):
    import oracle as O

    w, _, _ = O.select(conf.numpy(), C, lengths.numpy())
    return torch.from_numpy(w), None


def _worker(rank, world, port, B, k, C, seed, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2502_15197_b200.dist import dist_select

    g = torch.Generator().manual_seed(seed)
    conf_all = torch.rand(world * B, k, generator=g, dtype=torch.float64)
    conf_all[conf_all < 0.2] = 0.5  # ties across shards
    len_all = torch.randint(1, k + 1, (world * B,), generator=g, dtype=torch.int32)
    sl = slice(rank * B, (rank + 1) * B)
    res = dist_select(conf_all[sl].contiguous(), C, len_all[sl].contiguous(), select_fn=_oracle_select)
    ref, _ = _oracle_select(conf_all, C, len_all)
    ok = torch.equal(res.windows, ref[sl]) and res.row0 == rank * B
    ok = ok and int(res.win_offsets[-1]) == int(ref[sl].sum())
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("B,k,C", [(8, 4, 10), (50, 6, 77), (33, 3, 1)])
def test_two_rank_selection_equals_single_device(B, k, C):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, k, C, B * 31 + C, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
