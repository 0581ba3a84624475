"""Configuration-scale selection parity against goldens produced by the REFERENCE itself
(tests/golden/make_golden_scale.py ran tetris_sched's cumulative_products / select_tetris / expected_accepted on the
seeded matrices of tests/golden/scale_inputs.py: cfg1..cfg5 shapes, quantised ties with -0.0, ragged rows, the cfg4
capacity sweep C = 4096..65536, and B = 16384 x 16 at C = 131072).

CPU: the inputs regenerate bit-identically (sha256) and the C oracle reproduces every golden (windows, all four
PolicyStats, cum bits, expected_accepted).  GPU: the product selectors (select1 for <= 16384 cells, the grid selector
above) through ops.select, the exact heapq replay for `comparisons`, and the full TetrisStep's selection (selection +
accept test + sampler launches) reproduce them bit for bit."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))
from scale_inputs import conf_matrix, dec_windows, sha  # noqa: E402

GOLD = json.loads((HERE / "golden" / "select_scale.json").read_text())["cases"]
IDS = [f"{c['tag']}-C{c['C']}" for c in GOLD]


def _inputs(c):
    a, ln = conf_matrix(c["B"], c["k"], c["recipe"], c["seed"])
    assert sha(a) == c["conf_sha256"] and sha(ln) == c["lengths_sha256"], "input recipe no longer reproduces"
    return a, ln


def _cum_full(cum, ln):
    out = np.zeros_like(cum)
    mask = np.arange(cum.shape[1])[None, :] < ln[:, None]
    out[mask] = cum[mask]
    return out


@pytest.mark.parametrize("c", GOLD, ids=IDS)
def test_oracle_matches_reference_at_scale(c):
    import oracle as O

    a, ln = _inputs(c)
    w, cum, st = O.select(a, c["C"], ln)
    assert np.array_equal(w, dec_windows(c["windows"]))
    assert list(st) == c["stats"]
    assert sha(_cum_full(cum, ln)) == c["cum_sha256"]
    assert O.expected_accepted(a, w, ln) == float.fromhex(c["expected_accepted"])


@pytest.mark.gpu
@pytest.mark.parametrize("c", GOLD, ids=IDS)
def test_gpu_select_matches_reference_at_scale(c):
    import torch

    from paper_2502_15197_b200 import ops

    a, ln = _inputs(c)
    A = torch.from_numpy(a).cuda()
    L = torch.from_numpy(ln).cuda()
    res = ops.select(A, c["C"], L, want_cum=True)
    stats_exact = ops.heap_stats(res.cum, c["C"], L)
    ea = ops.expected_accepted(A, res.windows, L)
    ops.raise_for_status(res.status)
    w = res.windows.cpu().numpy()
    ref = dec_windows(c["windows"])
    assert np.array_equal(w, ref), f"windows differ at rows {np.nonzero(w != ref)[0][:10]}"
    assert sha(_cum_full(res.cum.cpu().numpy(), ln)) == c["cum_sha256"], "cum bits differ"
    st = res.stats.cpu().numpy()
    assert list(st[:3]) == c["stats"][:3], "closed-form extracts / inserts / peak_queue"
    assert list(stats_exact.cpu().numpy()) == c["stats"], "heapq replay (comparisons)"
    assert float(ea.item()) == float.fromhex(c["expected_accepted"])
    assert np.array_equal(np.diff(res.win_offsets.cpu().numpy()), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("c", GOLD, ids=IDS)
def test_step_selection_matches_reference_at_scale(c):
    """The selection inside the fused product step (tetris_select_accept_f32 + sampler launches), at a small V (the
    selection does not depend on V)."""
    import torch

    from paper_2502_15197_b200 import ops
    from paper_2502_15197_b200.synthetic import make_batch

    a, ln = _inputs(c)
    B, k, V = c["B"], c["k"], 256
    bt = make_batch(B, k, V, seed=c["seed"], device="cuda")
    step = ops.TetrisStep(B, k, V, c["C"], mode="stochastic", device="cuda")
    step.run(torch.from_numpy(a).cuda(), torch.from_numpy(ln).cuda(), bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    assert np.array_equal(step.windows.cpu().numpy(), dec_windows(c["windows"]))
    assert list(step.stats.cpu().numpy()[:3]) == c["stats"][:3]
