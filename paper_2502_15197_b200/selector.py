"""Drop-in for tetris_sched.selector's TETRIS path (selector.py:32-176, :286-306), computed on the GPU.

`cumulative_products` and `select_tetris` keep the reference's signatures and return this package's mirrors of the
reference dataclasses (Candidate, Selection, PolicyStats: same fields, same frozen equality).  The prefix products
and the global top-C selection run in `select_kernel`; PolicyStats.comparisons — a property of CPython's heapq
schedule — comes from the exact heap-replay kernel (disable with exact_stats=False to get -1 and skip it).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _types, ops
from .accept_model import AcceptanceMatrix, _device, matrix_to_device
from .errors import CapacityExceededError, OracleSizeExceededError  # noqa: F401  (re-exported names)

__all__ = ["Candidate", "Selection", "PolicyStats", "cumulative_products", "select_tetris", "expected_accepted",
           "select_tensor", "select_fixed_window", "select_dsd"]


@dataclass(frozen=True)
class Candidate:
    """One draftable token: request `row`, 1-based `depth`, cumulative acceptance `cum` (selector.py:32-39)."""

    row: int
    depth: int
    cum: float


@dataclass(frozen=True)
class Selection:
    """Prefix-closed selection stored as per-row window sizes (selector.py:42-82)."""

    windows: tuple

    def __post_init__(self) -> None:
        for i, w in enumerate(self.windows):
            if w < 0:
                raise ValueError(f"window for row {i} is negative: {w}")

    @property
    def size(self) -> int:
        return sum(self.windows)

    def pairs(self) -> set:
        return {(i, j) for i, w in enumerate(self.windows) for j in range(1, w + 1)}

    @classmethod
    def from_pairs(cls, pairs: Sequence, n_rows: int) -> "Selection":
        windows = [0] * n_rows
        seen = set(map(tuple, pairs))
        for i, j in seen:
            if not 0 <= i < n_rows:
                raise ValueError(f"row {i} outside 0..{n_rows - 1}")
            if j < 1:
                raise ValueError(f"depth {j} must be >= 1")
            windows[i] = max(windows[i], j)
        for i, w in enumerate(windows):
            for j in range(1, w + 1):
                if (i, j) not in seen:
                    raise ValueError(f"selection is not prefix-closed: row {i} has depth {w} but is missing depth {j}")
        return cls(tuple(windows))


@dataclass(frozen=True)
class PolicyStats:
    """Priority-queue accounting of one select_tetris call (selector.py:85-92)."""

    extracts: int
    inserts: int
    peak_queue: int
    comparisons: int


for _name, _cls in (("Candidate", Candidate), ("Selection", Selection), ("PolicyStats", PolicyStats)):
    _types.set_default(_name, _cls)


def cumulative_products(probs: AcceptanceMatrix) -> list:
    """Per-row candidates scored by the running product of acceptance rates (selector.py:95-110).  `probs` is any
    object with `.rows` (this package's AcceptanceMatrix or the reference's)."""
    a, ln = matrix_to_device(probs)
    res = ops.select(a, 0, ln, want_cum=True)
    ops.raise_for_status(res.status, "cumulative_products")
    cum = res.cum.cpu().numpy().tolist()
    cand = _types.get("Candidate")
    return [[cand(row=i, depth=j + 1, cum=cum[i][j]) for j in range(len(row))]
            for i, row in enumerate(probs.rows)]


def _pack_candidates(candidates) -> tuple:
    """Candidate lists -> dense [B, kmax] cum + lengths; like the reference, positions (not .row/.depth) count."""
    B = len(candidates)
    k = max((len(r) for r in candidates), default=0)
    vals = np.zeros((B, max(k, 1)), np.float64)
    ln = np.zeros(B, np.int32)
    for i, row in enumerate(candidates):
        ln[i] = len(row)
        if row:
            vals[i, : len(row)] = [c.cum for c in row]
    return vals, ln


def select_tetris(candidates: Sequence, capacity: int, *, exact_stats: bool = True) -> tuple:
    """Greedy capacity filling by cumulative acceptance probability (selector.py:133-176)."""
    if capacity < 0:
        raise ValueError(f"capacity must be >= 0, got {capacity}")
    B = len(candidates)
    sel_t, stats_t = _types.get("Selection"), _types.get("PolicyStats")
    if B == 0:
        return sel_t(()), stats_t(0, 0, 0, 0)
    vals, ln = _pack_candidates(candidates)
    if vals.shape[1] > ops.N.MAX_K:
        raise ValueError(f"rows deeper than {ops.N.MAX_K} candidates are not supported")
    dev = _device()
    v = torch.from_numpy(vals).to(dev)
    L = torch.from_numpy(ln).to(dev)
    res = ops.select(v, int(capacity), L, vals_are_cum=True)
    if exact_stats:
        st = ops.heap_stats(v, int(capacity), L).cpu().numpy()
    else:
        st = res.stats.cpu().numpy()
    ops.raise_for_status(res.status, "select_tetris")
    windows = tuple(int(x) for x in res.windows.cpu().numpy())
    return sel_t(windows), stats_t(int(st[0]), int(st[1]), int(st[2]), int(st[3]))


def select_fixed_window(n_rows: int, window: int, capacity: int) -> Selection:
    """Classic batched speculation: every row sends the same `window` tokens (selector.py:179-190)."""
    if n_rows < 1:
        raise ValueError(f"n_rows must be >= 1, got {n_rows}")
    if window < 0:
        raise ValueError(f"window must be >= 0, got {window}")
    if n_rows * window > capacity:
        raise CapacityExceededError(
            f"{n_rows} rows x window {window} = {n_rows * window} tokens exceeds capacity {capacity}")
    return _types.get("Selection")((window,) * n_rows)


def select_dsd(alpha_estimate: float, n_rows: int, capacity: int, depth_limit: int) -> Selection:
    """Adaptive common window from a scalar acceptance-rate estimate (selector.py:193-222)."""
    return _types.get("Selection")((ops.dsd_window(alpha_estimate, n_rows, capacity, depth_limit),) * n_rows)


def expected_accepted(selection: Selection, probs: AcceptanceMatrix) -> float:
    """Expected accepted draft tokens under `selection` (selector.py:286-306)."""
    if len(selection.windows) != len(probs.rows):
        raise ValueError(f"selection covers {len(selection.windows)} rows, matrix has {len(probs.rows)}")
    for window, row in zip(selection.windows, probs.rows):
        if window > len(row):
            raise ValueError(f"selection window {window} deeper than row of depth {len(row)}")
    a, ln = matrix_to_device(probs)
    w = torch.tensor(selection.windows, dtype=torch.int32, device=a.device)
    return float(ops.expected_accepted(a, w, ln).item())


def select_tensor(conf: torch.Tensor, capacity: int, lengths: torch.Tensor = None) -> ops.SelectResult:
    """Batched entry point: conf [B, k] f64 CUDA tensor of acceptance rates -> SelectResult (no host sync)."""
    return ops.select(conf, capacity, lengths)
