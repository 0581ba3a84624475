"""GPU: the drop-in adapters (same names / signatures / exceptions as tetris_sched) against the reference's own
golden vectors (tests/golden/, produced by the reference) and its unit-test cases, restated (reference test file:line
cited per test).  Everything below runs through the CUDA kernels via the C ABI."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2502_15197_b200.accept_model import (AcceptanceMatrix, DegenerateResidualError, TokenDistribution,
                                                residual_distribution, sample_emitted_token, verify_token)
from paper_2502_15197_b200.selector import (Candidate, PolicyStats, Selection, cumulative_products,
                                            expected_accepted, select_tetris)
from paper_2502_15197_b200.sim_engine import apply_verification, credit

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _f(xs):
    return [float.fromhex(x) for x in xs]


@pytest.fixture(scope="module")
def sel():
    return json.loads((G / "select.json").read_text())


@pytest.fixture(scope="module")
def tok():
    return json.loads((G / "token.json").read_text())


# ---- goldens --------------------------------------------------------------------------------------------------------
def test_golden_select(sel):
    for case in sel["monotone"]:
        m = AcceptanceMatrix.from_rows([_f(r) for r in case["rows"]])
        cands = cumulative_products(m)
        assert [[c.cum for c in r] for r in cands] == [_f(r) for r in case["cum"]], case["tag"]
        s, st = select_tetris(cands, case["capacity"])
        assert list(s.windows) == case["windows"], case["tag"]
        assert [st.extracts, st.inserts, st.peak_queue, st.comparisons] == case["stats"], case["tag"]
        assert expected_accepted(s, m) == float.fromhex(case["expected_accepted"]), case["tag"]


def test_golden_select_candidate_lists(sel):
    for case in sel["candidates"]:
        lists = [[Candidate(i, j + 1, c) for j, c in enumerate(_f(r))] for i, r in enumerate(case["cum"])]
        s, st = select_tetris(lists, case["capacity"])
        assert list(s.windows) == case["windows"]
        assert [st.extracts, st.inserts, st.peak_queue, st.comparisons] == case["stats"]


def test_golden_verify_token(tok):
    for c in tok["verify_token"]:
        ps, pm = TokenDistribution(_f(c["ps"])), TokenDistribution(_f(c["pm"]))
        assert verify_token(ps, pm, c["token"], float.fromhex(c["u"])) is c["accepted"]


def test_golden_residual(tok):
    for c in tok["residual"]:
        ps, pm = TokenDistribution(_f(c["ps"])), TokenDistribution(_f(c["pm"]))
        if c["residual"] is None:
            with pytest.raises(DegenerateResidualError):
                residual_distribution(ps, pm)
            continue
        np.testing.assert_allclose(residual_distribution(ps, pm).probs, _f(c["residual"]), rtol=1e-12, atol=1e-15)


def test_golden_sampled_chain(tok):
    """sample_emitted_token consumes the reference's uniforms in the reference's order and emits its token."""
    for c in tok["chain"][:60]:
        ps, pm = TokenDistribution(_f(c["ps"])), TokenDistribution(_f(c["pm"]))
        t, acc = sample_emitted_token(ps, pm, np.random.default_rng(c["seed"]))
        assert (t, acc) == (c["token"], c["accepted"])


def test_golden_apply_verification():
    for c in json.loads((G / "verify_matrix.json").read_text()):
        truth = AcceptanceMatrix.from_rows([_f(r) for r in c["rows"]])
        out = apply_verification(Selection(tuple(c["windows"])), truth, np.random.default_rng(c["seed"]))
        assert list(out) == c["accepted"]


# ---- the reference unit tests, restated ---------------------------------------------------------------------------
def test_cumprod_kats():  # test_selector.py:29-39
    cands = cumulative_products(AcceptanceMatrix.from_rows([[0.9, 0.9, 0.9], [0.5, 0.5]]))
    assert [c.cum for c in cands[0]] == pytest.approx([0.9, 0.81, 0.729])
    assert [(c.row, c.depth) for c in cands[1]] == [(1, 1), (1, 2)]
    assert [c.cum for c in cumulative_products(AcceptanceMatrix.from_rows([[0.5, 0.0, 0.8]]))[0]] == [0.5, 0.0, 0.0]


def test_select_kats():  # test_selector.py:51-85
    m = AcceptanceMatrix.from_rows([[0.9, 0.9, 0.9], [0.5, 0.5]])
    assert select_tetris(cumulative_products(m), 3)[0].windows == (3, 0)
    assert expected_accepted(Selection((3, 0)), m) == pytest.approx(2.439, abs=1e-12)
    assert select_tetris(cumulative_products(m), 4)[0].windows == (3, 1)
    eq = AcceptanceMatrix.from_rows([[0.7] * 3] * 2)
    assert select_tetris(cumulative_products(eq), 4)[0].windows == (2, 2)
    m2 = AcceptanceMatrix.from_rows([[0.9], [0.5]])
    s, st = select_tetris(cumulative_products(m2), 0)
    assert s.windows == (0, 0) and st.extracts == 0
    s, st = select_tetris(cumulative_products(m2), 10)
    assert s.windows == (1, 1) and st.extracts == 2
    z = AcceptanceMatrix.from_rows([[0.0, 0.0], [0.5]])
    assert select_tetris(cumulative_products(z), 3)[0].windows == (2, 1)
    t = AcceptanceMatrix.from_rows([[0.6] * 2] * 3)
    assert select_tetris(cumulative_products(t), 1)[0].windows == (1, 0, 0)
    with pytest.raises(ValueError):
        select_tetris([], -1)


def test_certificate_and_stats_random():  # test_selector.py:87-121
    rng = np.random.default_rng(29)
    for _ in range(60):
        n = int(rng.integers(1, 5))
        m = AcceptanceMatrix.from_rows([rng.random(int(rng.integers(1, 6))).tolist() for _ in range(n)])
        C = int(rng.integers(0, 9))
        cands = cumulative_products(m)
        s, st = select_tetris(cands, C)
        all_cums = sorted((c.cum for r in cands for c in r), reverse=True)
        picked = sorted((cands[i][j - 1].cum for i, w in enumerate(s.windows) for j in range(1, w + 1)), reverse=True)
        assert picked == all_cums[: min(C, len(all_cums))]
        assert st.extracts == s.size <= C and st.peak_queue <= m.n_rows and st.inserts <= s.size + m.n_rows
        assert select_tetris(cands, C) == (s, st)


@pytest.mark.parametrize("alpha", [0.1, 0.5, 0.9])
@pytest.mark.parametrize("n_rows,k", [(2, 1), (4, 2), (8, 4)])
def test_equal_rates_collapse(alpha, n_rows, k):  # test_selector.py:208-217
    m = AcceptanceMatrix.from_rows([[alpha] * (k + 2)] * n_rows)
    assert select_tetris(cumulative_products(m), n_rows * k)[0] == Selection((k,) * n_rows)


def test_verify_token_kats():  # test_accept_model.py:149-176
    assert verify_token(TokenDistribution([0.2, 0.8]), TokenDistribution([0.5, 0.5]), 0, 0.999) is True
    ps, pm = TokenDistribution([0.5, 0.5]), TokenDistribution([0.2, 0.8])
    assert verify_token(ps, pm, 0, 0.39) is True
    assert verify_token(ps, pm, 0, 0.41) is False
    p = TokenDistribution([0.25, 0.75])
    assert all(verify_token(p, p, 1, u) for u in (0.0, 0.5, 0.999))
    for args in ((ps, pm, 2, 0.5), (ps, pm, 0, 1.0), (ps, TokenDistribution([1.0]), 0, 0.5)):
        with pytest.raises(ValueError):
            verify_token(*args)


def test_residual_kats():  # test_accept_model.py:179-195
    r = residual_distribution(TokenDistribution([0.5, 0.5]), TokenDistribution([0.2, 0.8]))
    np.testing.assert_allclose(r.probs, [0.0, 1.0], atol=1e-12)
    r = residual_distribution(TokenDistribution([0.25, 0.25, 0.5]), TokenDistribution([0.5, 0.25, 0.25]))
    np.testing.assert_allclose(r.probs, [1.0, 0.0, 0.0], atol=1e-12)
    with pytest.raises(DegenerateResidualError):
        residual_distribution(TokenDistribution([0.3, 0.7]), TokenDistribution([0.3, 0.7]))


def test_sampled_chain_chi2():  # test_accept_model.py:244-257 (fewer draws: one GPU round trip per draw)
    rng = np.random.default_rng(123)
    ps, pm = TokenDistribution([0.6, 0.3, 0.1]), TokenDistribution([0.2, 0.3, 0.5])
    n = 3000
    counts = np.zeros(3)
    for _ in range(n):
        counts[sample_emitted_token(ps, pm, rng)[0]] += 1
    expected = n * pm.probs
    assert float(((counts - expected) ** 2 / expected).sum()) < 13.8


def test_apply_verification_cases():  # test_sim_engine.py:102-128
    truth = AcceptanceMatrix.from_rows([[1.0, 1.0], [0.0, 0.0]])
    assert apply_verification(Selection((2, 2)), truth, np.random.default_rng(0)) == (2, 0)
    casc = AcceptanceMatrix.from_rows([[1.0, 0.0, 1.0]])
    for seed in range(5):
        assert apply_verification(Selection((3,)), casc, np.random.default_rng(seed)) == (1,)
    with pytest.raises(ValueError):
        apply_verification(Selection((2,)), AcceptanceMatrix.from_rows([[0.5]]), np.random.default_rng(0))


def test_policy_isolation():  # test_sim_engine.py:208-233
    truth = AcceptanceMatrix.from_rows([[0.9, 1.0, 1.0], [0.2, 1.0, 1.0]])
    surrogate = AcceptanceMatrix.from_rows([[0.9] * 3, [0.2] * 3])
    sel1, _ = select_tetris(cumulative_products(surrogate), 4)
    acc1 = apply_verification(sel1, truth, np.random.default_rng(99))
    rows = [list(r) for r in truth.rows]
    for i, a in enumerate(acc1):
        if a < sel1.windows[i]:
            for j in range(a + 1, len(rows[i])):
                rows[i][j] = 1.0 - rows[i][j]
    acc2 = apply_verification(sel1, AcceptanceMatrix.from_rows(rows), np.random.default_rng(99))
    assert acc2 == acc1


def test_credit_cap():  # test_sim_engine.py:180-190
    assert credit((4, 4, 4, 4), (2, 2, 2, 2)) == (2, 2, 2, 2)
    assert credit((0, 3, 1), (5, 5, 1)) == (1, 4, 1)


def test_dataclass_contracts():  # test_selector.py:220-232
    assert Selection.from_pairs([(0, 1), (0, 2), (2, 1)], n_rows=3).windows == (2, 0, 1)
    with pytest.raises(ValueError):
        Selection.from_pairs([(0, 2)], n_rows=1)
    with pytest.raises(ValueError):
        Selection((1, -1))
    assert PolicyStats(1, 2, 3, 4) == PolicyStats(1, 2, 3, 4)
