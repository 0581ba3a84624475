"""GPU, world_size 2 on one device (gloo for the exchange): the full request-sharded TetrisStep — the all-gather of
scores, the global selection over both shards' rows, this rank's accept / resample / compaction — against the CPU
oracle of the whole batch.  (The production exchange is NCCL over NVLink; the kernels and the host logic are the
same.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, k, V, C, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        from paper_2502_15197_b200 import ops
        from paper_2502_15197_b200.synthetic import make_batch

        shards = [make_batch(B, k, V, seed=500 + r, ragged=True) for r in range(world)]  # every rank's inputs
        bt = shards[rank]
        step = ops.TetrisStep(B, k, V, C, group=dist.group.WORLD)
        step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
        torch.cuda.synchronize()
        ops.raise_for_status(step.status)
        conf_all = np.concatenate([s.conf.cpu().numpy() for s in shards])
        len_all = np.concatenate([s.lengths.cpu().numpy() for s in shards])
        w_ref, _, _ = O.select(conf_all, C, len_all)
        ok = np.array_equal(step.windows_all.cpu().numpy(), w_ref)
        wl = w_ref[rank * B:(rank + 1) * B]
        acc, tok, _ = O.verify_stochastic(bt.p.cpu().numpy(), bt.q.cpu().numpy(), bt.d.cpu().numpy(), wl,
                                          bt.u_acc.cpu().numpy(), bt.u_res.cpu().numpy(), nthreads=4)
        ok = ok and np.array_equal(step.accepted.cpu().numpy(), acc) and np.array_equal(step.out_tok.cpu().numpy(),
                                                                                        tok)
        off, toks = O.compact(acc, tok, bt.d.cpu().numpy())
        ok = ok and np.array_equal(step.offsets.cpu().numpy(), off)
        ok = ok and np.array_equal(step.tokens.cpu().numpy()[: off[-1]], toks)
        q.put((rank, bool(ok), ""))
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("B,k,V,C", [(300, 8, 4096, 2400), (1024, 16, 2048, 16384)])
def test_two_rank_tetris_step(B, k, V, C):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, k, V, C, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def _nccl_worker(port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
        from paper_2502_15197_b200.dist import gather_scores

        g = torch.Generator(device="cuda").manual_seed(5)
        conf = torch.rand(64, 7, dtype=torch.float64, device="cuda", generator=g)
        lens = torch.randint(0, 8, (64,), dtype=torch.int32, device="cuda", generator=g)
        conf_all = torch.zeros_like(conf)
        len_all = torch.zeros_like(lens)
        gather_scores(conf_all, len_all, conf, lens)  # the coalesced NCCL path (one group of two all-gathers)
        torch.cuda.synchronize()
        q.put(bool(torch.equal(conf_all, conf) and torch.equal(len_all, lens)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put(repr(e))


def test_nccl_coalesced_score_exchange():
    """The production exchange path (NCCL, coalesced all-gathers) runs and round-trips at world size 1 — the only NCCL
    world this one-GPU box can form."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    p.join(240)
    assert p.exitcode == 0
    assert q.get(timeout=5) is True
