"""GPU: the end-to-end host-buffer API (ops.HostTetrisStep) — p / q in pinned host memory, the needed rows moved by
DMA after the selection (staged) or read by the kernels through the mapping (zero-copy) — gives the device step's
results bit for bit, and the CPU oracle's."""
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
                                           ("greedy", "zero-copy")])
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
