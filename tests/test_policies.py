"""Baseline policies: select_fixed_window / select_dsd drop-ins (selector.py:179-222) and the
uniform-window tensor API + fixed-window step on the GPU."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2502_15197_b200 import ops
from paper_2502_15197_b200.errors import CapacityExceededError
from paper_2502_15197_b200.selector import Selection, select_dsd, select_fixed_window
from sim_step import dsd_window as oracle_dsd_window


# ---- host-side adapters: the reference's own known answers (test_selector.py:128-155) ------------------------------
def test_fixed_window_kats():
    sel = select_fixed_window(2, 2, 4)
    assert sel.windows == (2, 2)
    assert sel.pairs() == {(0, 1), (0, 2), (1, 1), (1, 2)}
    with pytest.raises(CapacityExceededError):
        select_fixed_window(2, 3, 4)
    with pytest.raises(ValueError):
        select_fixed_window(0, 1, 4)
    with pytest.raises(ValueError):
        select_fixed_window(2, -1, 4)


def test_dsd_kats():
    assert select_dsd(0.9, 2, 8, 4).windows == (4, 4)
    assert select_dsd(0.0, 2, 8, 4).windows == (1, 1)
    assert select_dsd(0.5, 4, 8, 8).windows == (2, 2, 2, 2)
    assert select_dsd(0.5, 4, 3, 8).windows == (0, 0, 0, 0)
    with pytest.raises(ValueError):
        select_dsd(1.5, 2, 8, 4)


def test_dsd_window_matches_restatement():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        a = float(rng.choice([0.0, 1.0, rng.random(), 1e-300, 1 - 1e-16]))
        n = int(rng.integers(1, 40))
        c = int(rng.integers(0, 400))
        d = int(rng.integers(1, 40))
        assert ops.dsd_window(a, n, c, d) == oracle_dsd_window(a, n, c, d)


# ---- device -------------------------------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("B,k,w", [(1, 1, 0), (7, 5, 3), (1024, 16, 8), (5000, 16, 20), (65535, 4, 2)])
def test_uniform_windows(B, k, w):
    g = torch.Generator().manual_seed(B)
    ln = torch.randint(0, k + 1, (B,), generator=g, dtype=torch.int32)
    win, off = ops.uniform_windows(w, ln.cuda())
    ref = np.minimum(w, ln.numpy())
    assert np.array_equal(win.cpu().numpy(), ref)
    assert np.array_equal(off.cpu().numpy(), np.concatenate([[0], np.cumsum(ref)]))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["stochastic", "greedy"])
def test_fixed_window_step_matches_oracle(mode):
    from paper_2502_15197_b200.synthetic import make_batch

    B, k, V, w = 300, 8, 4096, 3
    bt = make_batch(B, k, V, seed=5, ragged=True, mode=mode)
    step = ops.TetrisStep(B, k, V, B * w, mode=mode, policy="fixed")
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    wref = np.minimum(w, bt.lengths.cpu().numpy())
    assert np.array_equal(step.windows.cpu().numpy(), wref)
    p, d = bt.p.cpu().numpy(), bt.d.cpu().numpy()
    if mode == "stochastic":
        acc, tok, _ = O.verify_stochastic(p, bt.q.cpu().numpy(), d, wref, bt.u_acc.cpu().numpy(),
                                          bt.u_res.cpu().numpy(), nthreads=8)
    else:
        acc, tok = O.verify_greedy(p, d, wref, nthreads=8)
    assert np.array_equal(step.accepted.cpu().numpy(), acc)
    assert np.array_equal(step.out_tok.cpu().numpy(), tok)
    off, toks = O.compact(acc, tok, d)
    assert np.array_equal(step.offsets.cpu().numpy(), off)
    assert np.array_equal(step.tokens.cpu().numpy()[: off[-1]], toks)


@pytest.mark.gpu
def test_greedy_dominates_fixed_window():  # test_selector.py:193-205, through the GPU adapters
    from paper_2502_15197_b200.accept_model import AcceptanceMatrix
    from paper_2502_15197_b200.selector import cumulative_products, expected_accepted, select_tetris

    rng = np.random.default_rng(103)
    for _ in range(60):
        n = int(rng.integers(1, 5))
        rows = [list(rng.random(int(rng.integers(1, 5)))) for _ in range(n)]
        m = AcceptanceMatrix.from_rows(rows)
        kk = int(rng.integers(1, min(m.depths()) + 1))
        cap = m.n_rows * kk
        fixed = select_fixed_window(m.n_rows, kk, cap)
        greedy, _ = select_tetris(cumulative_products(m), cap)
        assert isinstance(greedy, Selection)
        assert expected_accepted(greedy, m) >= expected_accepted(fixed, m) - 1e-12
