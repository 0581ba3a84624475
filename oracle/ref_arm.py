"""The reference CPU path composed per step, for bench.py's CPU baseline and `--impl reference` arm.
TEST / BASELINE INFRASTRUCTURE ONLY: never imported by the product package.

The reference package (tetris_sched 0.1.0) is used ITSELF where it is installed (`baseline/_ref`, staged by
tests/ref_suite/stage.py; kind "reference"), else the line-by-line port oracle/reference_port.py (kind "port"):

  selection     AcceptanceMatrix.from_rows -> cumulative_products -> select_tetris   (selector.py:95-176)
  per request   verify_token at each selected depth until the first rejection      (accept_model.py:291-313)
                residual_distribution of the rejected depth's rows                 (accept_model.py:316-327)
                inverse CDF of Generator.choice with the request's uniform          (accept_model.py:364, :368)
                (all accepted: the bonus token from the target row at depth w)
  compaction    d[b, :a_b] ++ [x_b]                                                  (sim_engine.py:467-471)

TokenDistribution's 1e-9 sum check (accept_model.py:273-275) rejects fp32 softmax rows at V = 128256, so the
per-position distributions are built without re-validating (the same object, `.probs` set directly): verify_token
only reads two scalars of them, so they hold the fp32 rows (exact fp64 upcast on read); the two rows of a rejected
depth are upcast to fp64 before residual_distribution, as TokenDistribution's own constructor would.  Generator.choice
draws its uniform internally; the request's uniform is applied with the identical arithmetic
(cumsum / cdf[-1] / searchsorted 'right', reference_port.choice_index).

Verification fans out over requests two ways: one thread, and a fork-based `multiprocessing` pool on
all host cores (the pool is created once, outside the timed region, like a serving process would keep it).
"""
from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
sys.path.insert(0, str(HERE))
import reference_port as RP  # noqa: E402

_REF = None


def reference_modules():
    """(selector, accept_model) of tetris_sched from baseline/_ref, or None if it is not staged."""
    global _REF
    if _REF is None:
        path = ROOT / "baseline" / "_ref"
        try:
            if (path / "tetris_sched").exists() and str(path) not in sys.path:
                sys.path.insert(0, str(path))
            import tetris_sched.accept_model as A
            import tetris_sched.selector as S

            _REF = (S, A)
        except Exception:
            _REF = False
    return _REF or None


def kind() -> str:
    return "reference" if reference_modules() else "port"


# ---------------------------------------------------------------------------------------------------------------
def select(rows, C):
    """windows tuple of the reference's select_tetris(cumulative_products(AcceptanceMatrix.from_rows(rows)), C)."""
    ref = reference_modules()
    if ref:
        S, A = ref
        sel, _ = S.select_tetris(S.cumulative_products(A.AcceptanceMatrix.from_rows(rows)), C)
        return sel.windows
    return RP.select_tetris(RP.cumulative_products(rows), C)[0]


def _td(A, arr):
    td = A.TokenDistribution.__new__(A.TokenDistribution)
    td.probs = arr
    return td


def verify_request(p_rows, q_rows, d, w, u_acc, u_res, mode="stochastic"):
    """(accepted, emitted token) of one request through the reference's functions (see module docstring)."""
    if mode == "greedy":
        return RP.verify_request_greedy(p_rows, d, w)
    ref = reference_modules()
    if not ref:
        return RP.verify_request(p_rows, q_rows, d, w, u_acc, u_res)
    _, A = ref
    a = w
    for j in range(w):
        if not A.verify_token(_td(A, q_rows[j]), _td(A, p_rows[j]), int(d[j]), float(u_acc[j])):
            a = j
            break
    if a < w:
        res = A.residual_distribution(_td(A, np.asarray(q_rows[a], np.float64)),
                                      _td(A, np.asarray(p_rows[a], np.float64)))
        return a, RP.choice_index(res.probs, float(u_res))
    return a, RP.choice_index(np.asarray(p_rows[w], np.float64), float(u_res))


# ---------------------------------------------------------------------------------------------------------------
# fork-based pool: the host inputs are module globals set before the fork, so workers inherit them (no pickling)
_H = None
_W = None
_MODE = "stochastic"


def _work(span):
    lo, hi = span
    h = _H
    return [verify_request(h["p"][b], h["q"][b] if h.get("q") is not None else None, h["d"][b], _W[b],
                           h["u_acc"][b] if h.get("u_acc") is not None else None,
                           h["u_res"][b] if h.get("u_res") is not None else None, _MODE)
            for b in range(lo, hi)]


class ReferenceStep:
    """One reference step over host inputs h = {p [n, k+1, V], q [n, k, V], d, conf, lengths, u_acc, u_res} where
    the vocabulary rows cover the first n requests (the bounded verification sample) and the scalars all B."""

    def __init__(self, h, C, mode="stochastic", processes=None):
        self.h, self.C, self.mode = h, C, mode
        self.rows = [list(map(float, h["conf"][b, : h["lengths"][b]])) for b in range(h["conf"].shape[0])]
        self.processes = processes if processes is not None else (os.cpu_count() or 1)
        self.pool = None

    def start_pool(self):
        global _H, _MODE
        if self.pool is None and self.processes > 1:
            _H, _MODE = self.h, self.mode
            self.pool = mp.get_context("fork").Pool(self.processes)
        return self

    def close(self):
        if self.pool is not None:
            self.pool.terminate()
            self.pool = None

    def run(self, n, parallel):
        """Selection over all requests, then verification of requests [0, n).  Returns (select s, verify s,
        emitted tokens, [(accepted, token)])."""
        global _W
        t0 = time.perf_counter()
        windows = select(self.rows, self.C)
        t1 = time.perf_counter()
        _W = windows
        if parallel and self.pool is not None:
            step = -(-n // (self.processes * 4))
            spans = [(lo, min(n, lo + step)) for lo in range(0, n, step)]
            # the windows travel with each task (the pool forked before this step's selection)
            parts = self.pool.starmap_async(_work_with_windows, [(s, windows) for s in spans]).get(timeout=900)
            out = [r for part in parts for r in part]
        else:
            out = _work((0, n))
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1, sum(a + 1 for a, _ in out), out


def _work_with_windows(span, windows):
    global _W
    _W = windows
    return _work(span)


# ---------------------------------------------------------------------------------------------------------------
def numpy_agreement(p_rows, q_rows, residual, u_res, gpu_tok):
    """For each request: the token numpy's Generator.choice arithmetic draws from the row the GPU sampled (residual of
    (p_rows[b], q_rows[b]) or the bonus row p_rows[b]) with the request's uniform; returns the mismatch count."""
    from concurrent.futures import ThreadPoolExecutor

    def one(b):
        cdf = RP.numpy_cdf(p_rows[b], q_rows[b] if residual[b] else None)
        return int(RP.numpy_choice(cdf, float(u_res[b])))

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        ref = np.array(list(ex.map(one, range(len(u_res)))))
    return int(np.count_nonzero(ref != np.asarray(gpu_tok))), ref
