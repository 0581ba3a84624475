"""GPU: the end-to-end host-buffer API (ops.HostTetrisStep) — p / q in pinned host memory, the needed rows gathered
over the mapping into device memory after the selection (staged) or read by the streaming kernels through the mapping
(zero-copy) — gives the device step's results bit for bit, and the CPU oracle's."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2502_15197_b200 import ops
from paper_2502_15197_b200.synthetic import make_batch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("mode,transfer", [("stochastic", "staged"), ("stochastic", "zero-copy"),
                                           ("greedy", "staged"), ("greedy", "zero-copy")])
@pytest.mark.parametrize("B,k,V,C", [(64, 8, 16384, 200), (200, 5, 8200, 500), (40, 3, 1003, 60)])
def test_host_step_matches_device_step(mode, transfer, B, k, V, C):
    bt = make_batch(B, k, V, seed=B + k, mode=mode, ragged=True)
    dev_step = ops.TetrisStep(B, k, V, C, mode=mode)
    dev_step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    p_h = bt.p.cpu().pin_memory()
    q_h = bt.q.cpu().pin_memory() if mode == "stochastic" else None
    small = [t.cpu().pin_memory() for t in (bt.conf, bt.lengths, bt.d, bt.u_acc, bt.u_res)]
    hs = ops.HostTetrisStep(B, k, V, C, p_h, q_h, mode=mode, transfer=transfer)
    for _ in range(2):  # twice: the workspace counters are left at zero
        hs.run(*(small if mode == "stochastic" else small[:3]))
        torch.cuda.synchronize()
        n = int(hs.offsets_host[-1])
        assert np.array_equal(hs.offsets_host.numpy(), _np(dev_step.offsets))
        assert np.array_equal(hs.tokens_host.numpy()[:n], _np(dev_step.tokens)[:n])
        assert np.array_equal(hs.accepted_host.numpy(), _np(dev_step.accepted))
    ops.raise_for_status(hs.step.status)
    w_ref, _, _ = O.select(_np(bt.conf), C, _np(bt.lengths))
    if mode == "stochastic":
        acc_ref, tok_ref, _ = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), w_ref, _np(bt.u_acc),
                                                  _np(bt.u_res), None, nthreads=8)
    else:
        acc_ref, tok_ref = O.verify_greedy(_np(bt.p), _np(bt.d), w_ref, nthreads=8)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None)
    assert np.array_equal(hs.offsets_host.numpy(), off_ref)
    assert np.array_equal(hs.tokens_host.numpy()[: off_ref[-1]], toks_ref)


@pytest.mark.parametrize("mode", ["stochastic", "greedy"])
@pytest.mark.parametrize("transfer", ["staged", "zero-copy"])
def test_host_step_k0(mode, transfer):
    """k = 0 (nothing drafted): every request emits its bonus token; q_host may be None."""
    B, k, V, C = 32, 0, 4096, 10
    bt = make_batch(B, k, V, seed=3, mode=mode)
    dev_step = ops.TetrisStep(B, k, V, C, mode=mode)
    dev_step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    hs = ops.HostTetrisStep(B, k, V, C, bt.p.cpu().pin_memory(), None, mode=mode, transfer=transfer)
    small = [t.cpu().pin_memory() for t in (bt.conf, bt.lengths, bt.d, bt.u_acc, bt.u_res)]
    hs.run(*(small if mode == "stochastic" else small[:3]))
    torch.cuda.synchronize()
    ops.raise_for_status(hs.step.status)
    assert int(hs.offsets_host[-1]) == B
    assert np.array_equal(hs.tokens_host.numpy()[:B], _np(dev_step.tokens)[:B])


def test_pageable_host_inputs_are_registered_and_released():
    """tetris_map_host registers pageable memory itself; the mapping is released with the step."""
    from paper_2502_15197_b200 import _native as N

    B, k, V, C = 16, 4, 2048, 40
    bt = make_batch(B, k, V, seed=9)
    p_h, q_h = bt.p.cpu(), bt.q.cpu()  # pageable
    small = [t.cpu() for t in (bt.conf, bt.lengths, bt.d, bt.u_acc, bt.u_res)]
    hs = ops.HostTetrisStep(B, k, V, C, p_h, q_h, transfer="zero-copy")
    hs.run(*small)
    torch.cuda.synchronize()
    ops.raise_for_status(hs.step.status)
    ptr = p_h.data_ptr()
    del hs
    import gc

    gc.collect()
    # unregistered: mapping it again registers anew (would fail with cudaErrorHostMemoryAlreadyRegistered otherwise)
    dptr = N.map_host(ptr, p_h.numel() * 4)
    assert dptr != 0
    N.unmap_host(ptr)


@pytest.mark.parametrize("mode", ["stochastic", "greedy"])
def test_staged_host_step_in_cuda_graph(mode):
    """The staged host steps never synchronise the host, so a whole end-to-end step (H2D of the small inputs, the
    selection, the row gather, the verification, D2H of the results) replays from one CUDA graph."""
    B, k, V, C = 128, 8, 16384, 600
    bt = make_batch(B, k, V, seed=11, mode=mode, ragged=True)
    dev_step = ops.TetrisStep(B, k, V, C, mode=mode)
    dev_step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    p_h = bt.p.cpu().pin_memory()
    q_h = bt.q.cpu().pin_memory() if mode == "stochastic" else None
    small = [t.cpu().pin_memory() for t in (bt.conf, bt.lengths, bt.d, bt.u_acc, bt.u_res)]
    args = small if mode == "stochastic" else small[:3]
    hs = ops.HostTetrisStep(B, k, V, C, p_h, q_h, mode=mode, transfer="staged")
    assert hs.transfer == "staged"
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        hs.run(*args)
    torch.cuda.current_stream().wait_stream(cs)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        hs.run(*args)
    hs.offsets_host.zero_()
    hs.tokens_host.zero_()
    g.replay()
    torch.cuda.synchronize()
    n = int(hs.offsets_host[-1])
    assert n > 0 and np.array_equal(hs.offsets_host.numpy(), _np(dev_step.offsets))
    assert np.array_equal(hs.tokens_host.numpy()[:n], _np(dev_step.tokens)[:n])
