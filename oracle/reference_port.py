"""Pure-Python/numpy port of the reference's CPU algorithm for the hot path.  TEST INFRASTRUCTURE / CPU BASELINE ONLY.

/root/reference does not exist on the GPU box, so this restates the reference functions line by line (paths
relative to /root/reference/pkg/src/tetris_sched/) with the same numpy calls, and is what bench.py times as the
reference CPU implementation (`cpu_baseline.kind = "port"`, `--impl reference`):

  cumulative_products  selector.py:95-110   (sequential `cum *= alpha`)
  select_tetris        selector.py:133-176  (heapq over _HeapItem keys (-cum, row, depth), selector.py:113-130)
  verify_token         accept_model.py:291-313  (s <= m accept, else u < m / s)
  residual_distribution accept_model.py:316-327 (np.clip(pM - pS, 0); pairwise np.sum mass; diff / mass)
  Generator.choice     accept_model.py:364,368  (numpy: cdf = cumsum(p); cdf /= cdf[-1]; searchsorted(u, 'right'))
  apply_verification   sim_engine.py:374-404   (first rejection ends the row)
  credit / bonus       sim_engine.py:467-471, :407-409

TokenDistribution's 1e-9 sum check (accept_model.py:273-275) rejects fp32 softmax rows at V=128256, so the
verification here applies the identical arithmetic to the fp64-upcast rows directly.
"""
from __future__ import annotations

import heapq

import numpy as np


class _HeapItem:
    __slots__ = ("key", "row", "depth", "counter")

    def __init__(self, cum, row, depth, counter):
        self.key = (-cum, row, depth)
        self.row = row
        self.depth = depth
        self.counter = counter

    def __lt__(self, other):
        self.counter[0] += 1
        return self.key < other.key


def cumulative_products(rows):
    out = []
    for row in rows:
        cum = 1.0
        cands = []
        for alpha in row:
            cum *= alpha
            cands.append(cum)
        out.append(cands)
    return out


def select_tetris(cands, capacity):
    """Returns (windows tuple, (extracts, inserts, peak_queue, comparisons))."""
    if capacity < 0:
        raise ValueError(f"capacity must be >= 0, got {capacity}")
    n = len(cands)
    windows = [0] * n
    counter = [0]
    extracts = inserts = peak = 0
    if capacity > 0:
        heap = [_HeapItem(row[0], i, 1, counter) for i, row in enumerate(cands) if row]
        heapq.heapify(heap)
        inserts = peak = len(heap)
        while heap and extracts < capacity:
            item = heapq.heappop(heap)
            extracts += 1
            i, j = item.row, item.depth
            windows[i] = j
            if j < len(cands[i]):
                heapq.heappush(heap, _HeapItem(cands[i][j], i, j + 1, counter))
                inserts += 1
                peak = max(peak, len(heap))
    return tuple(windows), (extracts, inserts, peak, counter[0])


def choice_index(probs: np.ndarray, u: float) -> int:
    """numpy Generator.choice(V, p=probs) for a given uniform u (accept_model.py:364,368)."""
    cdf = np.cumsum(probs)
    cdf /= cdf[-1]
    return int(np.searchsorted(cdf, u, side="right"))


def verify_request(p_rows, q_rows, d, w, u_acc, u_res):
    """One request: p_rows [k+1, V], q_rows [k, V] (any float dtype), d [k], window w, uniforms.
    Returns (accepted, emitted token)."""
    a = w
    for j in range(w):
        t = int(d[j])
        s = float(q_rows[j][t])
        m = float(p_rows[j][t])
        if not (s <= m or float(u_acc[j]) < m / s):
            a = j
            break
    if a < w:
        diff = np.clip(np.asarray(p_rows[a], np.float64) - np.asarray(q_rows[a], np.float64), 0.0, None)
        mass = float(diff.sum())
        if mass <= 0.0:
            raise ValueError("degenerate residual")
        return a, choice_index(diff / mass, float(u_res))
    # bonus: Generator.choice(V, p=p[w]) on the fp64-upcast target row (choice normalises by its own cdf[-1])
    return a, choice_index(np.asarray(p_rows[w], np.float64), float(u_res))


def numpy_cdf(p_row, q_row=None) -> np.ndarray:
    """The CDF numpy's Generator.choice searches (accept_model.py:364,368): for a residual (q_row given) the
    probabilities are residual_distribution's `clip(p - q, 0) / pairwise-sum` (accept_model.py:316-327); for a bonus
    row the fp64-upcast target row itself.  cdf = cumsum(p); cdf /= cdf[-1]."""
    p64 = np.asarray(p_row, np.float64)
    if q_row is not None:
        diff = np.clip(p64 - np.asarray(q_row, np.float64), 0.0, None)
        mass = float(diff.sum())
        if mass <= 0.0:
            raise ValueError("degenerate residual")
        p64 = diff / mass
    cdf = np.cumsum(p64)
    cdf /= cdf[-1]
    return cdf


def numpy_choice(cdf: np.ndarray, u) -> np.ndarray:
    """searchsorted(cdf, u, 'right') for one or many uniforms (Generator.choice's inverse CDF)."""
    return np.searchsorted(cdf, u, side="right")


def verify_request_greedy(p_rows, d, w):
    for j in range(w + 1):
        am = int(np.argmax(p_rows[j]))
        if j == w or am != int(d[j]):
            return j, am
    raise AssertionError


def compact(accepted, out_tok, d, cap=None):
    toks = []
    offsets = [0]
    for b, a in enumerate(accepted):
        n = a + 1 if cap is None else min(a + 1, cap[b])
        seq = list(d[b][:a]) + [out_tok[b]]
        toks.extend(int(x) for x in seq[:n])
        offsets.append(len(toks))
    return offsets, toks
