"""CPU: pin the oracle (C restatement + numpy reference port) against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  No GPU needed."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import reference_port as RP

G = Path(__file__).resolve().parent / "golden"


def _f(xs):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


@pytest.fixture(scope="module")
def sel():
    return json.loads((G / "select.json").read_text())


@pytest.fixture(scope="module")
def tok():
    return json.loads((G / "token.json").read_text())


def _dense(rows):
    B = len(rows)
    k = max([len(r) for r in rows] + [1])
    a = np.zeros((B, k))
    ln = np.zeros(B, np.int32)
    for i, r in enumerate(rows):
        a[i, : len(r)] = _f(r)
        ln[i] = len(r)
    return a, ln


def test_select_matches_reference_exactly(sel):
    for case in sel["monotone"]:
        a, ln = _dense(case["rows"])
        w, cum, st = O.select(a, case["capacity"], ln)
        assert list(w) == case["windows"], case["tag"]
        assert list(st) == case["stats"], case["tag"]  # incl. heapq comparisons
        for i, r in enumerate(case["cum"]):
            assert np.array_equal(cum[i, : len(r)].view(np.uint64), _f(r).view(np.uint64))
        ea = O.expected_accepted(a, w)
        assert ea == float.fromhex(case["expected_accepted"])


def test_select_candidate_lists_match_reference(sel):
    for case in sel["candidates"]:
        a, ln = _dense(case["cum"])
        w, _, st = O.select(a, case["capacity"], ln, vals_are_cum=True)
        assert list(w) == case["windows"]
        assert list(st) == case["stats"]


def test_reference_port_select_matches_reference(sel):
    for case in sel["monotone"][:200] + []:
        rows = [list(_f(r)) for r in case["rows"]]
        w, st = RP.select_tetris(RP.cumulative_products(rows), case["capacity"])
        assert list(w) == case["windows"] and list(st) == case["stats"]


def test_verify_token_rule(tok):
    for c in tok["verify_token"]:
        assert O.verify_token(_f(c["ps"]), _f(c["pm"]), c["token"], float.fromhex(c["u"])) == c["accepted"]


def test_residual_within_tolerance(tok):
    """Oracle residual vs residual_distribution: same formula, mass summed in the contract's fixed fp64 tree
    instead of numpy's pairwise order -> |rel diff| <= 1e-12 (fp64 tolerance of the path)."""
    for c in tok["residual"]:
        ps, pm = _f(c["ps"]), _f(c["pm"])
        out, mass, rc = O.residual(ps, pm)
        if c["residual"] is None:
            assert rc == 2
            continue
        assert rc == 0
        np.testing.assert_allclose(out, _f(c["residual"]), rtol=1e-12, atol=1e-15)


def test_emitted_law_from_oracle_residual(tok):
    """emitted_law (accept_model.py:339-354) recomposed from the oracle residual reproduces the reference law."""
    for c in tok["residual"]:
        if "emitted_law" not in c:
            continue
        ps, pm = _f(c["ps"]), _f(c["pm"])
        acc = np.minimum(ps, pm)
        rej = 1.0 - float(acc.sum())
        if rej <= 0.0:
            law = acc
        else:
            out, _, rc = O.residual(ps, pm)
            law = acc + rej * out
        np.testing.assert_allclose(law, _f(c["emitted_law"]), rtol=0, atol=1e-12)
        assert 0.5 * np.abs(law - pm).sum() < 1e-12  # lossless (test_accept_model.py:226-237)


def test_sampler_matches_numpy_choice(tok):
    """The contract sampler draws numpy Generator.choice's index for the same uniform (reference goldens)."""
    agree = 0
    for c in tok["choice"]:
        idx, mass = O.sample(_f(c["p"]), float.fromhex(c["u"]))
        agree += idx == c["index"]
        assert RP.choice_index(_f(c["p"]), float.fromhex(c["u"])) == c["index"]
    assert agree == len(tok["choice"])


def test_sampled_chain_matches_reference(tok):
    """sample_emitted_token (accept_model.py:357-368) recomposed from oracle pieces with the same three uniforms."""
    for c in tok["chain"]:
        ps, pm = _f(c["ps"]), _f(c["pm"])
        u = _f(c["u"])
        t, _ = O.sample(ps, u[0])
        if O.verify_token(ps, pm, t, u[1]):
            got = (t, True)
        else:
            got = (O.sample(pm, u[2], q=ps)[0], False)
        assert got == (c["token"], c["accepted"])


def test_verify_matrix_matches_reference():
    cases = json.loads((G / "verify_matrix.json").read_text())
    for c in cases:
        a, ln = _dense(c["rows"])
        draws = _f(c["draws"]) if c["draws"] else np.zeros(1)
        acc = O.verify_matrix(a, np.array(c["windows"], np.int32), draws)
        assert list(acc) == c["accepted"]
        # the flat-stream contract: numpy's per-row rng.random(w) calls == one rng.random(sum w)
        assert np.array_equal(np.random.default_rng(c["seed"]).random(sum(c["windows"])), _f(c["draws"]))


def test_sampler_hierarchy_edge_cases():
    # single positive element anywhere, zero rows, u -> 1
    for V in (1, 7, 256, 8192, 8193, 20000):
        for pos in {0, V // 2, V - 1}:
            p = np.zeros(V)
            p[pos] = 0.3
            for u in (0.0, 0.5, np.nextafter(1.0, 0.0)):
                assert O.sample(p, u)[0] == pos
    assert O.sample(np.zeros(10), 0.5)[0] == -1
    rng = np.random.default_rng(0)
    for V in (3, 300, 9000, 40000):
        p = rng.dirichlet(np.ones(V) * 0.1)
        for u in rng.random(50):
            assert O.sample(p, u)[0] == RP.choice_index(p, u)


def test_compact_and_greedy_small():
    acc = np.array([0, 2, 1], np.int32)
    tok = np.array([7, 8, 9], np.int32)
    d = np.array([[1, 2], [3, 4], [5, 6]], np.int32)
    off, toks = O.compact(acc, tok, d)
    assert list(off) == [0, 1, 4, 6] and list(toks) == [7, 3, 4, 8, 5, 9]
    off, toks = O.compact(acc, tok, d, cap=np.array([5, 1, 1], np.int32))
    assert list(off) == [0, 1, 2, 3] and list(toks) == [7, 3, 5]
    p = np.zeros((1, 3, 5), np.float32)
    p[0, 0, 2] = 1.0
    p[0, 1, 4] = 1.0
    p[0, 2, 1] = 1.0
    a, t = O.verify_greedy(p, np.array([[2, 3]], np.int32), np.array([2], np.int32))
    assert (a[0], t[0]) == (1, 4)
