"""Drop-in for tetris_sched.accept_model's token-level API (accept_model.py:262-368), computed on the GPU.

Same names, argument meaning, return types and exceptions as the reference.  The containers (AcceptanceMatrix,
TokenDistribution) validate on construction exactly like the reference (host-side metadata checks); every
probability computation — the accept rule, the residual distribution and its mass, inverse-CDF sampling — runs in
the sm_100a kernels behind the C ABI.  Sampling follows the fixed-hierarchy contract of include/tetris_b200.h, which
draws the same index as numpy's Generator.choice for the same uniform up to last-bit rounding of the CDF.
"""
from __future__ import annotations

import math
import weakref
from collections import OrderedDict
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _types, ops
from .errors import DegenerateResidualError

__all__ = ["AcceptanceMatrix", "TokenDistribution", "DegenerateResidualError", "verify_token",
           "residual_distribution", "sample_emitted_token", "verify_tokens_batch", "matrix_to_device"]


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2502_15197_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class AcceptanceMatrix:
    """Conditional acceptance probabilities, one row per request (accept_model.py:37-70)."""

    rows: tuple

    def __post_init__(self) -> None:
        if not self.rows:
            raise ValueError("acceptance matrix needs at least one row")
        for i, row in enumerate(self.rows):
            if not row:
                raise ValueError(f"row {i} is empty; every row needs depth >= 1")
            for j, alpha in enumerate(row):
                if not 0.0 <= alpha <= 1.0:
                    raise ValueError(f"alpha[{i}][{j}] = {alpha!r} outside [0, 1]")

    @classmethod
    def from_rows(cls, rows: Iterable[Iterable[float]]) -> "AcceptanceMatrix":
        return cls(tuple(tuple(float(a) for a in row) for row in rows))

    @property
    def n_rows(self) -> int:
        return len(self.rows)

    def depths(self) -> tuple:
        return tuple(len(row) for row in self.rows)

    def to_device(self, device=None):
        """Dense [B, k] f64 (zero padded) + lengths [B] i32 on the GPU."""
        return matrix_to_device(self, device)


def matrix_to_device(matrix, device=None):
    """Any object with `.rows` (this package's AcceptanceMatrix or tetris_sched's) -> dense [B, k] f64 (zero padded)
    + lengths [B] i32 on the GPU."""
    rows = matrix.rows
    dev = device or _device()
    k = max((len(r) for r in rows), default=0)
    a = np.zeros((len(rows), max(k, 1)), np.float64)
    for i, r in enumerate(rows):
        a[i, : len(r)] = r
    ln = np.array([len(r) for r in rows], np.int32)
    return torch.from_numpy(a).to(dev), torch.from_numpy(ln).to(dev)


class TokenDistribution:
    """Probability vector over a finite vocabulary (accept_model.py:262-281)."""

    __slots__ = ("probs",)

    def __init__(self, probs) -> None:
        arr = np.array(probs, dtype=np.float64)
        if arr.ndim != 1 or arr.size < 1:
            raise ValueError("distribution must be a non-empty 1-d vector")
        if np.any(arr < 0.0):
            raise ValueError("distribution entries must be >= 0")
        total = float(arr.sum())
        if not math.isclose(total, 1.0, rel_tol=0.0, abs_tol=1e-9):
            raise ValueError(f"distribution sums to {total!r}, expected 1 within 1e-9")
        arr.setflags(write=False)
        self.probs = arr

    @property
    def vocab_size(self) -> int:
        return int(self.probs.size)


for _name, _cls in (("AcceptanceMatrix", AcceptanceMatrix), ("TokenDistribution", TokenDistribution),
                   ("DegenerateResidualError", DegenerateResidualError)):
    _types.set_default(_name, _cls)


def _check_pair(p_draft: TokenDistribution, p_target: TokenDistribution) -> None:
    if p_draft.vocab_size != p_target.vocab_size:
        raise ValueError(
            f"vocabulary mismatch: draft {p_draft.vocab_size} vs target {p_target.vocab_size}")


_row_cache: "OrderedDict[int, tuple]" = OrderedDict()
_ROW_CACHE_MAX = 64


def _device_row(arr, dev) -> torch.Tensor:
    """[1, V] f64 device copy of a distribution's probability vector.  Read-only vectors (TokenDistribution marks
    them so, accept_model.py:276) are immutable, so their device copy is cached by identity (a weak reference
    guards against id reuse): Monte Carlo callers that verify 10^6 tokens against one pair copy it once."""
    if isinstance(arr, np.ndarray) and not arr.flags.writeable:
        hit = _row_cache.get(id(arr))
        if hit is not None and hit[0]() is arr and hit[1].device == dev:
            _row_cache.move_to_end(id(arr))
            return hit[1]
        t = torch.from_numpy(np.array(arr, np.float64)).view(1, -1).to(dev)
        _row_cache[id(arr)] = (weakref.ref(arr), t)
        if len(_row_cache) > _ROW_CACHE_MAX:
            _row_cache.popitem(last=False)
        return t
    return torch.from_numpy(np.array(arr, np.float64)).view(1, -1).to(dev)


def _rows(*dists: TokenDistribution):
    dev = _device()
    return [_device_row(d.probs, dev) for d in dists]


def verify_token(p_draft: TokenDistribution, p_target: TokenDistribution, token: int, u: float) -> bool:
    """Exact accept/reject decision for one drafted token (accept_model.py:291-313)."""
    _check_pair(p_draft, p_target)
    if not 0 <= token < p_draft.vocab_size:
        raise ValueError(f"token {token} outside vocabulary of size {p_draft.vocab_size}")
    if not 0.0 <= u < 1.0:
        raise ValueError(f"u must lie in [0, 1), got {u!r}")
    ps, pt = _rows(p_draft, p_target)
    dev = ps.device
    acc = ops.verify_tokens(ps, pt, torch.tensor([int(token)], dtype=torch.int32, device=dev),
                            torch.tensor([float(u)], dtype=torch.float64, device=dev))
    return bool(int(acc[0].item()))


def verify_tokens_batch(p_draft: torch.Tensor, p_target: torch.Tensor, tokens: torch.Tensor,
                        u: torch.Tensor) -> torch.Tensor:
    """Batched verify_token over R (draft row, target row, token, u) tuples already on the GPU."""
    return ops.verify_tokens(p_draft, p_target, tokens, u)


def residual_distribution(p_draft: TokenDistribution, p_target: TokenDistribution) -> TokenDistribution:
    """Renormalised positive part of (target - draft) (accept_model.py:316-327)."""
    _check_pair(p_draft, p_target)
    ps, pt = _rows(p_draft, p_target)
    out, mass, st = ops.residual(ps, pt)
    try:
        ops.raise_for_status(st, "residual_distribution")  # DegenerateResidualError when the mass is 0
    except DegenerateResidualError as e:
        raise _types.get("DegenerateResidualError")(str(e)) from None
    return _types.get("TokenDistribution")(out[0].cpu().numpy())


def _sample(dist_row: torch.Tensor, u: float, q_row: torch.Tensor = None) -> int:
    dev = dist_row.device
    rows = torch.zeros(1, dtype=torch.int64, device=dev)
    idx, mass, st = ops.sample_rows(dist_row, rows, torch.tensor([u], dtype=torch.float64, device=dev), q=q_row,
                                    q_row=None if q_row is None else rows)
    ops.raise_for_status(st, "sample")
    return int(idx[0].item())


def sample_emitted_token(p_draft: TokenDistribution, p_target: TokenDistribution,
                         rng: np.random.Generator) -> tuple:
    """One pass through draft -> verify -> residual resample (accept_model.py:357-368); consumes the same uniforms
    from `rng` as the reference (one per choice, one for the accept test)."""
    _check_pair(p_draft, p_target)
    ps, pt = _rows(p_draft, p_target)
    token = _sample(ps, float(rng.random()))
    if verify_token(p_draft, p_target, token, float(rng.random())):
        return token, True
    return _sample(pt, float(rng.random()), q_row=ps), False
