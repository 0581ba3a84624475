"""Drop-in for the hot-path pieces of tetris_sched.sim_engine: apply_verification (sim_engine.py:374-404), the bonus
count (:407-409) and the per-request credit `min(acc + 1, remaining)` (:467-471), computed on the GPU.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import ops
from .accept_model import AcceptanceMatrix, _device
from .selector import Selection

__all__ = ["apply_verification", "bonus_tokens", "credit"]


def apply_verification(selection: Selection, truth: AcceptanceMatrix, rng: np.random.Generator) -> tuple:
    """Cascading accept/reject per row.  Consumes exactly windows[i] uniforms for row i, in row order, as
    `rng.random(sum(windows))` (identical stream to the reference's per-row `rng.random(w_i)` calls)."""
    if len(selection.windows) != truth.n_rows:
        raise ValueError(f"selection covers {len(selection.windows)} rows, truth has {truth.n_rows}")
    for window, row in zip(selection.windows, truth.rows):
        if window > len(row):
            raise ValueError(f"selection window {window} deeper than drafted depth {len(row)}")
    n = sum(selection.windows)
    draws = rng.random(n) if n else np.zeros(0)
    a, ln = truth.to_device()
    dev = a.device
    w = torch.tensor(selection.windows, dtype=torch.int32, device=dev)
    off = torch.zeros(len(selection.windows) + 1, dtype=torch.int32, device=dev)
    off[1:] = torch.cumsum(w, 0, dtype=torch.int32)
    u = torch.from_numpy(np.ascontiguousarray(draws if n else np.zeros(1), np.float64)).to(dev)
    acc = ops.verify_matrix(a, w, off, u, ln)
    return tuple(int(x) for x in acc.cpu().numpy())


def bonus_tokens(state) -> int:
    """Verification emits one extra token per request beyond the accepted run (sim_engine.py:407-409)."""
    return len(state.active)


def credit(accepted: Sequence[int], remaining: Sequence[int]) -> tuple:
    """Per-request credited tokens min(acc + 1, remaining) (sim_engine.py:467-471), via the compaction kernel."""
    dev = _device()
    acc = torch.tensor(list(accepted), dtype=torch.int32, device=dev)
    cap = torch.tensor(list(remaining), dtype=torch.int32, device=dev)
    B = acc.shape[0]
    d = torch.zeros(B, max(1, max(accepted, default=0)), dtype=torch.int32, device=dev)  # token ids are irrelevant
    tok = torch.zeros(B, dtype=torch.int32, device=dev)
    offsets, _ = ops.compact(acc, tok, d, cap)
    return tuple(int(x) for x in torch.diff(offsets).cpu().numpy())
