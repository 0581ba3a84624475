"""Drop-in for the hot-path pieces of tetris_sched.sim_engine: apply_verification (sim_engine.py:374-404), the bonus
count (:407-409) and the per-request credit `min(acc + 1, remaining)` (:467-471), computed on the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from . import ops
from .accept_model import AcceptanceMatrix, _device, matrix_to_device
from .selector import Selection

__all__ = ["apply_verification", "bonus_tokens", "credit", "GpuSimulator", "GpuStepOutcome"]


def apply_verification(selection: Selection, truth: AcceptanceMatrix, rng: np.random.Generator) -> tuple:
    """Cascading accept/reject per row.  Consumes exactly windows[i] uniforms for row i, in row order, as
    `rng.random(sum(windows))` (identical stream to the reference's per-row `rng.random(w_i)` calls)."""
    if len(selection.windows) != len(truth.rows):
        raise ValueError(f"selection covers {len(selection.windows)} rows, truth has {len(truth.rows)}")
    for window, row in zip(selection.windows, truth.rows):
        if window > len(row):
            raise ValueError(f"selection window {window} deeper than drafted depth {len(row)}")
    n = sum(selection.windows)
    draws = rng.random(n) if n else np.zeros(0)
    a, ln = matrix_to_device(truth)
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


# ---------------------------------------------------------------------------------------------------------------
# GPU-resident simulator step
# ---------------------------------------------------------------------------------------------------------------
POLICY_CODES = {"tetris": 0, "sd": 1, "dsd": 2}


@dataclass(frozen=True)
class GpuStepOutcome:
    """The observable fields of StepOutcome (sim_engine.py:278-295) produced on the device for one step."""

    step: int
    windows: tuple
    accepted: tuple
    credited: tuple
    bonus: int
    expected_accepted: float
    stats: object  # PolicyStats (tetris, with the exact heapq comparison count) or None
    completions: tuple  # ((request id, arrival step), ...) in active-list order
    alpha_hat: float
    tau: float = 0.0  # step wall time under the configured pipeline (sim_engine.py:412-425)

    @property
    def sent(self) -> int:
        return sum(self.windows)


class GpuSimulator:
    """run_step (sim_engine.py:454-495) with the batch state resident on the GPU.

    The draft phase stays with the caller (the draft model / acceptance source produces the truth and surrogate rows
    for the depths `depths()` reports, sim_engine.py:338-346); everything after it — policy windows, the cascade over
    the verify uniform stream, expected_accepted, credit, the DSD estimate and refill_batch — runs in
    tetris_select_f64 (tetris) + tetris_sim_step.  `uniforms` is the verify generator's stream (the reference draws
    rng.random(w_i) per row in order, i.e. one flat stream, sim_engine.py:393-396) and `lengths` the target-length
    stream: the first batch_size entries are the initial batch (init_state, :311-330), the rest feed refill_batch in
    completion order."""

    def __init__(self, batch_size: int, k: int, capacity: int, *, extra: int = 0, policy: str = "tetris",
                 dsd_decay: float = 0.9, dsd_initial_estimate: float = 0.5, uniforms=None, lengths=None, device=None,
                 pipeline: str = "sequential", draft_time_per_token: float = 0.0025,
                 selection_overhead: float = 0.0003, verify_time: float = 0.025, exact_stats: bool = True):
        if pipeline not in ("sequential", "parallel"):
            raise ValueError(f"pipeline must be 'sequential' or 'parallel', got {pipeline!r}")
        self.pipeline, self.draft_time_per_token = pipeline, draft_time_per_token
        self.selection_overhead, self.verify_time = selection_overhead, verify_time
        if policy not in POLICY_CODES:
            raise ValueError(f"policy must be one of {tuple(POLICY_CODES)}, got {policy!r}")
        if batch_size < 1 or batch_size > 1024:
            raise ValueError(f"batch_size must lie in [1, 1024], got {batch_size}")
        dev = _device() if device is None else torch.device(device)
        self.B, self.k, self.K, self.C, self.policy = batch_size, k, k + extra, int(capacity), policy
        self.dsd_decay = float(dsd_decay)
        lengths = np.ascontiguousarray(lengths, dtype=np.int32)
        if lengths.shape[0] < batch_size:
            raise ValueError("the length stream must cover the initial batch")
        self.uniforms = torch.from_numpy(np.array(uniforms, dtype=np.float64)).to(dev)
        self.lengths = torch.from_numpy(lengths[batch_size:].copy() if lengths.shape[0] > batch_size
                                        else np.ones(1, np.int32)).to(dev)
        self.n_lengths = max(0, lengths.shape[0] - batch_size)
        B = batch_size
        self.ids = torch.arange(B, dtype=torch.int64, device=dev)
        self.target = torch.from_numpy(lengths[:B].copy()).to(dev)
        self.served = torch.zeros(B, dtype=torch.int32, device=dev)
        self.arrival = torch.zeros(B, dtype=torch.int32, device=dev)
        self.alpha_hat = torch.tensor([dsd_initial_estimate], dtype=torch.float64, device=dev)
        self.counters = torch.tensor([0, 0, B, 0, 0, 0, 0], dtype=torch.int64, device=dev)
        self.windows = torch.zeros(B, dtype=torch.int32, device=dev)
        self.accepted = torch.zeros(B, dtype=torch.int32, device=dev)
        self.credited = torch.zeros(B, dtype=torch.int32, device=dev)
        self.expected = torch.zeros(1, dtype=torch.float64, device=dev)
        self.done_ids = torch.zeros(B, dtype=torch.int64, device=dev)
        self.done_arrival = torch.zeros(B, dtype=torch.int32, device=dev)
        self.depths_dev = torch.clamp(self.target, max=self.K).to(torch.int32)
        self.status = ops.new_status(dev)
        self.device = dev
        # exact_stats: PolicyStats.comparisons from the exact heapq replay (tetris_heap_stats_f64, one thread: the
        # count is a property of the sequential schedule); False takes the selection's closed forms and reports
        # comparisons = -1, which keeps the whole step parallel
        self.exact_stats = bool(exact_stats)
        # every per-step result comes back in ONE round of async copies into pinned buffers, then one stream sync
        self._host = {name: torch.empty(t.shape, dtype=t.dtype).pin_memory() for name, t in (
            ("counters", self.counters), ("windows", self.windows), ("accepted", self.accepted),
            ("credited", self.credited), ("expected", self.expected), ("alpha_hat", self.alpha_hat),
            ("done_ids", self.done_ids), ("done_arrival", self.done_arrival), ("depths", self.depths_dev),
            ("stats", torch.zeros(4, dtype=torch.int64)), ("status", self.status))}
        self._host["depths"].copy_(self.depths_dev)

    def depths(self) -> tuple:
        """Draft depths of the next step, min(k + extra, remaining) per active request (sim_engine.py:343); fetched
        with the previous step's results (no extra device round trip)."""
        return tuple(int(x) for x in self._host["depths"].numpy())

    def step(self, truth, surrogate=None) -> GpuStepOutcome:
        """One simulator step given the draft phase's truth (and surrogate) rows, ragged lists or [B, K] arrays whose
        row lengths are the current depths."""
        B, K, dev = self.B, self.K, self.device
        depths = self.depths()
        tr = self._pack(truth, depths)
        lens = torch.tensor(depths, dtype=torch.int32, device=dev)
        stats_t = None
        if self.policy == "tetris":
            sg = self._pack(truth if surrogate is None else surrogate, depths)
            res = ops.select(sg, self.C, lens, want_cum=self.exact_stats)
            self.windows.copy_(res.windows)
            # exact PolicyStats incl. heapq comparisons, or the selection's closed forms (comparisons -1)
            stats_t = ops.heap_stats(res.cum, self.C, lens) if self.exact_stats else res.stats
        N.call("tetris_sim_step", tr.data_ptr(), lens.data_ptr(), B, K, POLICY_CODES[self.policy], self.k, self.C,
               self.dsd_decay, self.uniforms.data_ptr(), self.uniforms.numel(), self.lengths.data_ptr(),
               self.n_lengths, self.windows.data_ptr(), self.ids.data_ptr(), self.target.data_ptr(),
               self.served.data_ptr(), self.arrival.data_ptr(), self.alpha_hat.data_ptr(), self.counters.data_ptr(),
               self.accepted.data_ptr(), self.credited.data_ptr(), self.expected.data_ptr(), self.done_ids.data_ptr(),
               self.done_arrival.data_ptr(), self.depths_dev.data_ptr(), self.status.data_ptr(),
               torch.cuda.current_stream(dev).cuda_stream)
        h = self._host
        for name, t in (("counters", self.counters), ("windows", self.windows), ("accepted", self.accepted),
                        ("credited", self.credited), ("expected", self.expected), ("alpha_hat", self.alpha_hat),
                        ("done_ids", self.done_ids), ("done_arrival", self.done_arrival), ("depths", self.depths_dev),
                        ("status", self.status)):
            h[name].copy_(t, non_blocking=True)
        if stats_t is not None:
            h["stats"].copy_(stats_t, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        ops.raise_for_status(h["status"], "sim step")
        cnt = h["counters"].numpy()
        n_done = int(cnt[4])
        stats = None
        if self.policy == "tetris":
            from .selector import PolicyStats

            st = h["stats"].numpy()
            stats = PolicyStats(int(st[0]), int(st[1]), int(st[2]), int(st[3]))
        comps = tuple(zip((int(x) for x in h["done_ids"].numpy()[:n_done]),
                          (int(x) for x in h["done_arrival"].numpy()[:n_done])))
        return GpuStepOutcome(
            tau=self.step_time(depths),
            step=int(cnt[3]) - 1,
            windows=tuple(int(x) for x in h["windows"].numpy()),
            accepted=tuple(int(x) for x in h["accepted"].numpy()),
            credited=tuple(int(x) for x in h["credited"].numpy()),
            bonus=B,
            expected_accepted=float(h["expected"].numpy()[0]),
            stats=stats,
            completions=comps,
            alpha_hat=float(h["alpha_hat"].numpy()[0]),
        )

    def step_time(self, drafted_depths) -> float:
        """step_time (sim_engine.py:412-425): drafting + selection, then verification (sequential) or the slower of
        the two (parallel)."""
        draft_path = self.draft_time_per_token * (max(drafted_depths) if drafted_depths else 0) + \
            self.selection_overhead
        if self.pipeline == "sequential":
            return draft_path + self.verify_time
        return max(draft_path, self.verify_time)

    def _pack(self, rows, depths) -> torch.Tensor:
        B, K = self.B, self.K
        if isinstance(rows, torch.Tensor):
            return rows.to(self.device, torch.float64).contiguous()
        if isinstance(rows, np.ndarray) and rows.ndim == 2:
            return torch.from_numpy(np.ascontiguousarray(rows, np.float64)).to(self.device)
        if hasattr(rows, "rows"):  # an AcceptanceMatrix
            rows = rows.rows
        out = np.zeros((B, K), np.float64)
        if len(rows) != B:
            raise ValueError(f"expected {B} rows, got {len(rows)}")
        for i, (r, d) in enumerate(zip(rows, depths)):
            if len(r) != d:
                raise ValueError(f"row {i} has {len(r)} entries, the draft depth is {d}")
            out[i, :d] = r
        return torch.from_numpy(out).to(self.device)
