"""Batched tensor API of the TETRIS hot path (CUDA tensors in, CUDA tensors out, stream-ordered, no host sync).

Every function launches the sm_100a kernels of libtetris_b200.so through the C ABI on the current torch stream.
Inputs must already be CUDA tensors; there is no CPU path.  Data-dependent errors are accumulated in a device status
word; call `raise_for_status(status)` (one host sync) where the reference would have raised.

Shapes (dense, row-major): conf/alpha/cum [B, k] f64, lengths [B] i32, p [B, k+1, V] f32 (target incl. the bonus
position), q [B, k, V] f32 (draft), d [B, k] i32 (draft tokens), u_acc [B, k] (dense) or [sum(windows)] (packed)
f64, u_res [B] f64.
"""
from __future__ import annotations

import os

from dataclasses import dataclass
from typing import Optional

import torch

from . import _native as N
from .errors import DegenerateResidualError

_I32 = torch.int32
_I64 = torch.int64
_F64 = torch.float64
_F32 = torch.float32


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream_handle(stream: Optional[torch.cuda.Stream] = None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _need_cuda(name: str, t: Optional[torch.Tensor], dtype, ndim: Optional[int] = None, optional=False):
    if t is None:
        if optional:
            return None
        raise ValueError(f"{name} is required")
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-d, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


class Workspace:
    """Caller-owned scratch for the kernels (zeroed once; kernels leave the arrival counters at zero).

    One workspace must not be used by two streams concurrently."""

    def __init__(self, device, op: int, B: int, k: int, V: int):
        self.nbytes = max(N.workspace_bytes(op, B, k, V), 256)
        self.buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=device)
        self.key = (op, B, k, V)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()


_ws_cache: dict = {}


def workspace(device, op: int, B: int, k: int, V: int, stream: Optional[torch.cuda.Stream] = None) -> Workspace:
    dev = torch.device(device)
    sh = _stream_handle(stream) if dev.type == "cuda" else 0
    key = (dev, sh, op)
    ws = _ws_cache.get(key)
    need = N.workspace_bytes(op, B, k, V)
    if ws is None or ws.nbytes < need:
        ws = Workspace(dev, op, B, k, V)
        _ws_cache[key] = ws
    return ws


def new_status(device) -> torch.Tensor:
    return torch.zeros(1, dtype=_I32, device=device)


def raise_for_status(status: torch.Tensor, context: str = "") -> None:
    """Host sync: map device status bits to the reference's exceptions."""
    s = int(status.item()) & 0xFFFFFFFF
    if not s:
        return
    where = f" ({context})" if context else ""
    if s & N.ST_BAD_TOKEN:
        raise ValueError(f"draft token outside the vocabulary{where}")
    if s & N.ST_BAD_UNIFORM:
        raise ValueError(f"uniform draw outside [0, 1){where}")
    if s & N.ST_BAD_WINDOW:
        raise ValueError(f"selection window deeper than the drafted row{where}")
    if s & N.ST_BAD_VALUE:
        raise ValueError(f"acceptance value outside [0, 1] or NaN{where}")
    if s & N.ST_STREAM_EXHAUSTED:
        raise ValueError(f"uniform or target-length stream exhausted{where}")
    if s & N.ST_DEGENERATE:
        raise DegenerateResidualError(f"target never rejects the draft; there is no residual to sample{where}")
    raise RuntimeError(f"unknown status bits {s:#x}{where}")


# ---------------------------------------------------------------------------------------------------------------
# stages (1)+(2): selection
# ---------------------------------------------------------------------------------------------------------------
@dataclass
class SelectResult:
    windows: torch.Tensor            # [B] i32
    win_offsets: torch.Tensor        # [B+1] i32, exclusive scan of windows
    stats: torch.Tensor              # [4] i64: extracts, inserts, peak_queue, comparisons (-1 unless exact)
    status: torch.Tensor             # [1] i32 device status bits
    cum: Optional[torch.Tensor] = None  # [B, k] f64 (when requested)


def select(vals: torch.Tensor, capacity: int, lengths: Optional[torch.Tensor] = None, *, vals_are_cum: bool = False,
           want_cum: bool = False, out: Optional[SelectResult] = None,
           stream: Optional[torch.cuda.Stream] = None) -> SelectResult:
    """cumulative_products + select_tetris (selector.py:95-176) on the GPU."""
    vals = _need_cuda("vals", vals, _F64, 2)
    B, k = vals.shape
    lengths = _need_cuda("lengths", lengths, _I32, 1, optional=True)
    if capacity < 0:
        raise ValueError(f"capacity must be >= 0, got {capacity}")
    dev = vals.device
    if out is None:
        out = SelectResult(
            windows=torch.empty(B, dtype=_I32, device=dev),
            win_offsets=torch.empty(B + 1, dtype=_I32, device=dev),
            stats=torch.empty(4, dtype=_I64, device=dev),
            status=new_status(dev),
            cum=torch.zeros(B, k, dtype=_F64, device=dev) if want_cum else None,
        )
    ws = workspace(dev, N.OP_ALL, B, k, 1, stream)
    N.call("tetris_select_f64", _ptr(vals), _ptr(lengths), B, k, int(capacity), int(bool(vals_are_cum)),
           _ptr(out.windows), _ptr(out.win_offsets), _ptr(out.cum), _ptr(out.stats), _ptr(out.status),
           ws.ptr, ws.nbytes, _stream_handle(stream))
    return out


def dsd_window(alpha_estimate: float, n_rows: int, capacity: int, depth_limit: int) -> int:
    """select_dsd's common window (selector.py:193-222): argmax over k in [1, min(depth_limit, capacity // n_rows)] of
    sum_{j<=k} alpha^j with the same fp64 running product / sum, first maximum wins; 0 when no token per row fits."""
    if not 0.0 <= alpha_estimate <= 1.0:
        raise ValueError(f"alpha_estimate {alpha_estimate!r} outside [0, 1]")
    if n_rows < 1:
        raise ValueError(f"n_rows must be >= 1, got {n_rows}")
    if depth_limit < 1:
        raise ValueError(f"depth_limit must be >= 1, got {depth_limit}")
    k_max = min(depth_limit, capacity // n_rows)
    if k_max < 1:
        return 0
    best_k, best, value, power = 1, alpha_estimate, alpha_estimate, alpha_estimate
    for k in range(2, k_max + 1):
        power *= alpha_estimate
        value += power
        if value > best:
            best, best_k = value, k
    return best_k


def uniform_windows(window: int, lengths: Optional[torch.Tensor] = None, B: Optional[int] = None, k: int = 0, *,
                    windows: Optional[torch.Tensor] = None, win_offsets: Optional[torch.Tensor] = None,
                    device=None, stream: Optional[torch.cuda.Stream] = None):
    """Baseline policies on the tensor API: windows[b] = min(window, lengths[b]) (fixed window / sd / dsd common
    window clamped to each drafted depth, sim_engine.py:358-368) and their exclusive scan, on the device."""
    if window < 0:
        raise ValueError(f"window must be >= 0, got {window}")
    lengths = _need_cuda("lengths", lengths, _I32, 1, optional=True)
    if lengths is not None:
        B = lengths.shape[0]
        device = lengths.device
    if B is None:
        raise ValueError("give lengths or B")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if windows is None:
        windows = torch.empty(B, dtype=_I32, device=dev)
    if win_offsets is None:
        win_offsets = torch.empty(B + 1, dtype=_I32, device=dev)
    N.call("tetris_uniform_windows", _ptr(lengths), B, k, int(window), _ptr(windows), _ptr(win_offsets),
           _stream_handle(stream))
    return windows, win_offsets


def heap_stats(cum: torch.Tensor, capacity: int, lengths: Optional[torch.Tensor] = None,
               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Exact PolicyStats incl. heapq comparisons (selector.py:151-176); single-thread accounting kernel."""
    cum = _need_cuda("cum", cum, _F64, 2)
    B, k = cum.shape
    lengths = _need_cuda("lengths", lengths, _I32, 1, optional=True)
    stats = torch.empty(4, dtype=_I64, device=cum.device)
    ws = workspace(cum.device, N.OP_ALL, B, k, 1, stream)
    N.call("tetris_heap_stats_f64", _ptr(cum), _ptr(lengths), B, k, int(capacity), _ptr(stats), ws.ptr, ws.nbytes,
           _stream_handle(stream))
    return stats


def expected_accepted(alpha: torch.Tensor, windows: torch.Tensor, lengths: Optional[torch.Tensor] = None,
                      status: Optional[torch.Tensor] = None) -> torch.Tensor:
    alpha = _need_cuda("alpha", alpha, _F64, 2)
    B, k = alpha.shape
    windows = _need_cuda("windows", windows, _I32, 1)
    out = torch.empty((), dtype=_F64, device=alpha.device)
    st = status if status is not None else new_status(alpha.device)
    N.call("tetris_expected_accepted_f64", _ptr(alpha), _ptr(lengths), _ptr(windows), B, k, _ptr(out), _ptr(st),
           _stream_handle())
    if status is None:
        raise_for_status(st, "expected_accepted")
    return out


# ---------------------------------------------------------------------------------------------------------------
# stage (3): verification
# ---------------------------------------------------------------------------------------------------------------
def verify_matrix(alpha: torch.Tensor, windows: torch.Tensor, win_offsets: torch.Tensor, u: torch.Tensor,
                  lengths: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None) -> torch.Tensor:
    """apply_verification (sim_engine.py:374-404) with the flat uniform stream u[win_offsets[b] + j]."""
    alpha = _need_cuda("alpha", alpha, _F64, 2)
    B, k = alpha.shape
    windows = _need_cuda("windows", windows, _I32, 1)
    win_offsets = _need_cuda("win_offsets", win_offsets, _I32, 1)
    u = _need_cuda("u", u, _F64, 1)
    lengths = _need_cuda("lengths", lengths, _I32, 1, optional=True)
    acc = torch.empty(B, dtype=_I32, device=alpha.device)
    st = status if status is not None else new_status(alpha.device)
    N.call("tetris_verify_matrix_f64", _ptr(alpha), _ptr(lengths), _ptr(windows), _ptr(win_offsets), _ptr(u), B, k,
           _ptr(acc), _ptr(st), _stream_handle())
    if status is None:
        raise_for_status(st, "apply_verification")
    return acc


def verify_tokens(p_draft: torch.Tensor, p_target: torch.Tensor, token: torch.Tensor, u: torch.Tensor,
                  status: Optional[torch.Tensor] = None) -> torch.Tensor:
    """verify_token (accept_model.py:291-313) for R (draft row, target row, token, u) tuples; rows [R, V] f64."""
    p_draft = _need_cuda("p_draft", p_draft, _F64, 2)
    p_target = _need_cuda("p_target", p_target, _F64, 2)
    if p_draft.shape != p_target.shape:
        raise ValueError(f"vocabulary mismatch: draft {tuple(p_draft.shape)} vs target {tuple(p_target.shape)}")
    R, V = p_draft.shape
    token = _need_cuda("token", token, _I32, 1)
    u = _need_cuda("u", u, _F64, 1)
    acc = torch.empty(R, dtype=_I32, device=p_draft.device)
    st = status if status is not None else new_status(p_draft.device)
    N.call("tetris_verify_tokens_f64", _ptr(p_draft), _ptr(p_target), _ptr(token), _ptr(u), R, V, _ptr(acc), _ptr(st),
           _stream_handle())
    if status is None:
        raise_for_status(st, "verify_token")
    return acc


@dataclass
class VerifyResult:
    accepted: torch.Tensor  # [B] i32
    out_tok: torch.Tensor   # [B] i32 (correction or bonus token)
    status: torch.Tensor    # [1] i32
    mass: Optional[torch.Tensor] = None  # [B] f64 (stochastic, when requested)


def verify_stochastic(p: torch.Tensor, q: torch.Tensor, d: torch.Tensor, windows: torch.Tensor,
                      u_acc: torch.Tensor, u_res: torch.Tensor, win_offsets: Optional[torch.Tensor] = None, *,
                      want_mass: bool = False, out: Optional[VerifyResult] = None,
                      stream: Optional[torch.cuda.Stream] = None) -> VerifyResult:
    p = _need_cuda("p", p, _F32, 3)
    q = _need_cuda("q", q, _F32, 3)
    B, k1, V = p.shape
    k = k1 - 1
    if tuple(q.shape) != (B, k, V):
        raise ValueError(f"q must be [B, k, V] = {(B, k, V)}, got {tuple(q.shape)}")
    d = _need_cuda("d", d, _I32, 2)
    windows = _need_cuda("windows", windows, _I32, 1)
    u_acc = _need_cuda("u_acc", u_acc, _F64)
    u_res = _need_cuda("u_res", u_res, _F64, 1)
    win_offsets = _need_cuda("win_offsets", win_offsets, _I32, 1, optional=True)
    dev = p.device
    if out is None:
        out = VerifyResult(torch.empty(B, dtype=_I32, device=dev), torch.empty(B, dtype=_I32, device=dev),
                           new_status(dev), torch.empty(B, dtype=_F64, device=dev) if want_mass else None)
    ws = workspace(dev, N.OP_VERIFY, B, k, V, stream)
    N.call("tetris_verify_stochastic_f32", _ptr(p), _ptr(q), _ptr(d), _ptr(windows), _ptr(win_offsets),
           _ptr(u_acc), _ptr(u_res), B, k, V, _ptr(out.accepted), _ptr(out.out_tok), _ptr(out.mass),
           _ptr(out.status), ws.ptr, ws.nbytes, _stream_handle(stream))
    return out


def verify_greedy(p: torch.Tensor, d: torch.Tensor, windows: torch.Tensor, *, out: Optional[VerifyResult] = None,
                  stream: Optional[torch.cuda.Stream] = None) -> VerifyResult:
    p = _need_cuda("p", p, _F32, 3)
    B, k1, V = p.shape
    k = k1 - 1
    d = _need_cuda("d", d, _I32, 2)
    windows = _need_cuda("windows", windows, _I32, 1)
    dev = p.device
    if out is None:
        out = VerifyResult(torch.empty(B, dtype=_I32, device=dev), torch.empty(B, dtype=_I32, device=dev),
                           new_status(dev))
    ws = workspace(dev, N.OP_VERIFY, B, k, V, stream)
    N.call("tetris_verify_greedy_f32", _ptr(p), _ptr(d), _ptr(windows), B, k, V, _ptr(out.accepted),
           _ptr(out.out_tok), _ptr(out.status), ws.ptr, ws.nbytes, _stream_handle(stream))
    return out


def sample_rows(p: torch.Tensor, p_row: torch.Tensor, u: torch.Tensor, q: Optional[torch.Tensor] = None,
                q_row: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None):
    """Sample one index per (p row[, q row]) pair under the sampling contract; p/q are [rows, V] f32 or f64."""
    if p.dtype not in (_F32, _F64):
        raise ValueError("p must be float32 or float64")
    p = _need_cuda("p", p, p.dtype, 2)
    V = p.shape[1]
    q = _need_cuda("q", q, p.dtype, 2, optional=True)
    p_row = _need_cuda("p_row", p_row, _I64, 1)
    R = p_row.shape[0]
    q_row = _need_cuda("q_row", q_row, _I64, 1, optional=True)
    u = _need_cuda("u", u, _F64, 1)
    dev = p.device
    idx = torch.empty(R, dtype=_I32, device=dev)
    mass = torch.empty(R, dtype=_F64, device=dev)
    st = status if status is not None else new_status(dev)
    ws = workspace(dev, N.OP_VERIFY, R, 0, V)
    fn = "tetris_sample_rows_f64" if p.dtype == _F64 else "tetris_sample_rows_f32"
    N.call(fn, _ptr(p), _ptr(q), _ptr(p_row), _ptr(q_row), _ptr(u), R, V, _ptr(idx), _ptr(mass), _ptr(st), ws.ptr,
           ws.nbytes, _stream_handle())
    return idx, mass, st


def residual(p_draft: torch.Tensor, p_target: torch.Tensor, status: Optional[torch.Tensor] = None):
    """residual_distribution (accept_model.py:316-327) for R row pairs [R, V] f64 -> ([R, V] f64, mass [R])."""
    p_draft = _need_cuda("p_draft", p_draft, _F64, 2)
    p_target = _need_cuda("p_target", p_target, _F64, 2)
    if p_draft.shape != p_target.shape:
        raise ValueError(f"vocabulary mismatch: draft {tuple(p_draft.shape)} vs target {tuple(p_target.shape)}")
    R, V = p_draft.shape
    dev = p_draft.device
    out = torch.empty(R, V, dtype=_F64, device=dev)
    mass = torch.empty(R, dtype=_F64, device=dev)
    st = status if status is not None else new_status(dev)
    ws = workspace(dev, N.OP_VERIFY, R, 0, V)
    N.call("tetris_residual_f64", _ptr(p_draft), _ptr(p_target), R, V, _ptr(out), _ptr(mass), _ptr(st), ws.ptr,
           ws.nbytes, _stream_handle())
    return out, mass, st


def probs_from_logits(z: torch.Tensor, lse: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The logits contract materialised (include/tetris_b200.h): prob(z, lse) for bf16 logits z [..., V] and their
    row log-sum-exp lse [...] f32 -> fp32 [..., V]."""
    if not isinstance(z, torch.Tensor) or not z.is_cuda or z.dtype != torch.bfloat16 or not z.is_contiguous():
        raise ValueError("z must be a contiguous bfloat16 CUDA tensor")
    lse = _need_cuda("lse", lse, _F32)
    V = z.shape[-1]
    R = z.numel() // max(V, 1)
    if lse.numel() != R:
        raise ValueError(f"lse must hold one value per row ({R}), got {lse.numel()}")
    if out is None:
        out = torch.empty(z.shape, dtype=_F32, device=z.device)
    N.call("tetris_probs_from_logits_bf16", z.data_ptr(), lse.data_ptr(), R, V, out.data_ptr(), _stream_handle())
    return out


# ---------------------------------------------------------------------------------------------------------------
# stage (4): compaction
# ---------------------------------------------------------------------------------------------------------------
def compact(accepted: torch.Tensor, out_tok: torch.Tensor, d: torch.Tensor, cap: Optional[torch.Tensor] = None, *,
            offsets: Optional[torch.Tensor] = None, tokens: Optional[torch.Tensor] = None,
            stream: Optional[torch.cuda.Stream] = None):
    """Emitted tokens d[b,:a_b] ++ [x_b] (capped by cap[b]) packed back to back; returns (offsets[B+1], tokens)."""
    accepted = _need_cuda("accepted", accepted, _I32, 1)
    out_tok = _need_cuda("out_tok", out_tok, _I32, 1)
    d = _need_cuda("d", d, _I32, 2)
    cap = _need_cuda("cap", cap, _I32, 1, optional=True)
    B, k = d.shape
    dev = d.device
    if offsets is None:
        offsets = torch.empty(B + 1, dtype=_I32, device=dev)
    if tokens is None:
        tokens = torch.empty(B * (k + 1), dtype=_I32, device=dev)
    N.call("tetris_compact", _ptr(accepted), _ptr(out_tok), _ptr(d), _ptr(cap), B, k, _ptr(offsets), _ptr(tokens),
           _stream_handle(stream))
    return offsets, tokens


# ---------------------------------------------------------------------------------------------------------------
# one full verification step with preallocated buffers (CUDA-graph capturable)
# ---------------------------------------------------------------------------------------------------------------
SPEC_MAX_REQUESTS = 4096  # tetris_resample_spec_f32's limit (per call, local rows) on a full B200; a device with
# fewer SMs takes min(4096, 32 x SMs) (tetris_spec_max_requests, queried per TetrisStep)
# below this much streaming the early start does not pay (csrc/verify.cu kSpecMinChunks); env override for A/B runs
SPEC_MIN_CHUNKS = int(os.environ.get("TETRIS_SPEC_MIN_CHUNKS", "4096"))
_NO_SPEC = os.environ.get("TETRIS_NO_SPEC") == "1"  # A/B timing switch: the plain sampler
FUSED_MAX_CELLS = 2048  # csrc/launch.h kFusedMaxCells: the one-launch stochastic step up to this many cells
FUSED_MAX_ROWS = 4096   # ... and this many selected rows (kFusedMaxRpt * 512: the fused scans' rows per thread)
_NO_FUSED = "TETRIS_NO_FUSED" in os.environ  # A/B timing switch: the two-launch step (read by the library too)


class TetrisStep:
    """select -> verify (stochastic or greedy) -> compact for fixed shapes; every launch goes on the current stream,
    all buffers are preallocated, nothing synchronises the host, so `run` can be captured in a CUDA graph."""

    def __init__(self, B: int, k: int, V: int, capacity: int, mode: str = "stochastic", device="cuda",
                 u_layout: str = "dense", group=None, policy: str = "tetris", shard=None):
        if mode not in ("stochastic", "greedy"):
            raise ValueError(f"mode must be 'stochastic' or 'greedy', got {mode!r}")
        if policy not in ("tetris", "fixed"):
            raise ValueError(f"policy must be 'tetris' or 'fixed', got {policy!r}")
        if policy == "fixed" and group is not None:
            raise ValueError("the fixed-window baseline needs no global exchange; run it per shard without a group")
        self.policy = policy
        self.B, self.k, self.V, self.C, self.mode = B, k, V, int(capacity), mode
        self.u_layout = u_layout
        dev = torch.device(device)
        self.device = dev
        # request-sharded selection: gather every shard's scores, select globally, keep the local slice (dist.py)
        self.group = group
        self.world, self.rank = 1, 0
        if group is not None:
            import torch.distributed as dist

            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        elif shard is not None:
            # (world, rank) without a process group: the caller hands run() the already gathered [world*B, k] scores
            # and lengths (single-GPU measurement of one rank's share of a sharded step)
            self.world, self.rank = int(shard[0]), int(shard[1])
            if not 0 <= self.rank < self.world:
                raise ValueError(f"shard rank {self.rank} outside world {self.world}")
        Bg = B * self.world
        self.Bg = Bg
        # NCCL groups: the exchange and the step are ONE native call (tetris_dist_step_*, csrc/dist.cu) on the
        # torch communicator; other backends (gloo tests) gather in Python (dist.gather_scores)
        self._comm = None
        self._gathered_len = self._exchanged = False
        if group is not None:
            from .dist import nccl_comm

            self._comm = nccl_comm(group, dev)
        if self.world > 1 or group is not None:
            if u_layout != "dense":
                raise ValueError("sharded steps use the dense uniform layout")
            self.conf_all = torch.zeros(Bg, k, dtype=_F64, device=dev)
            self.len_all = torch.zeros(Bg, dtype=_I32, device=dev)
        self.windows_all = torch.zeros(Bg, dtype=_I32, device=dev)
        self.windows = self.windows_all[self.rank * B:(self.rank + 1) * B]
        self.win_offsets = torch.zeros(Bg + 1, dtype=_I32, device=dev)
        self.stats = torch.zeros(4, dtype=_I64, device=dev)
        self.status = new_status(dev)
        self.accepted = torch.zeros(B, dtype=_I32, device=dev)
        self.out_tok = torch.zeros(B, dtype=_I32, device=dev)
        self.mass = torch.zeros(B, dtype=_F64, device=dev)
        self.offsets = torch.zeros(B + 1, dtype=_I32, device=dev)
        self.tokens = torch.zeros(B * (k + 1), dtype=_I32, device=dev)
        self.ws = Workspace(dev, N.OP_ALL, Bg, k, V)
        self._lib = N.load()
        with torch.cuda.device(dev):
            self.spec_max = min(SPEC_MAX_REQUESTS, N.spec_max_requests())

    def exchange(self, conf, lengths=None) -> None:
        """Issue the sharded step's only exchange -- every rank's scores and drafted depths all-gathered into this
        step's conf_all / len_all -- NOW, on the current stream; then call run(..., gathered=True), which skips it.
        The exchange needs only the draft phase's confidences, so a serving loop issues it as soon as drafting ends
        (e.g. on a side stream, before the target model's forward pass that produces p) and takes it off the
        verification step's critical path.  NCCL: tetris_dist_gather_scores on the torch communicator."""
        if self.group is None:
            raise ValueError("exchange() needs the step's process group")
        self._gathered_len = lengths is not None
        self._exchanged = True
        if self._comm is not None:
            self._check(self._lib.tetris_dist_gather_scores(
                conf.data_ptr(), _ptr(lengths), self.B, self.k, self._comm, self.conf_all.data_ptr(),
                _ptr(self.len_all if lengths is not None else None), torch.cuda.current_stream().cuda_stream))
        else:
            from .dist import gather_scores

            ln = lengths if lengths is not None else torch.full((self.B,), self.k, dtype=_I32, device=conf.device)
            gather_scores(self.conf_all, self.len_all, conf, ln, self.group)
            self._gathered_len = True

    def run(self, conf, lengths, p, q, d, u_acc=None, u_res=None, cap=None, events=None, window=None,
            gathered: bool = False) -> None:
        """events: optional 4 torch.cuda.Events recorded around select / verify / compact (kernel timing).  The
        stochastic step is two launches (select+accept+compaction offsets, then the streaming sampler), so its
        events bracket [select kernel | sampler | nothing].  gathered=True: exchange() already gathered the scores
        (conf / lengths are then not read)."""
        lib, ws, s = self._lib, self.ws, torch.cuda.current_stream().cuda_stream
        B, k, V = self.B, self.k, self.V
        if events is not None:
            events[0].record()
        if self.policy == "fixed":
            self._run_fixed(lengths, p, q, d, u_acc, u_res, cap, events, window)
            return
        if gathered:  # exchange() already issued the all-gather on this stream
            if self.group is None or not self._exchanged:
                raise ValueError("gathered=True needs the step's process group and a prior exchange()")
            self._exchanged = False  # one exchange per step
            sel_conf, sel_len = self.conf_all, (self.len_all if self._gathered_len else None)
        elif self._comm is not None and events is None and self._dist_native(p, q):
            self._run_dist(conf, lengths, p, q, d, u_acc, u_res, cap)
            return
        elif self.world > 1 and self.group is not None:
            from .dist import gather_scores

            gather_scores(self.conf_all, self.len_all, conf, lengths, self.group)  # one coalesced NCCL exchange
            sel_conf, sel_len = self.conf_all, self.len_all
        else:  # world 1, or a shard given the gathered scores directly
            sel_conf, sel_len = conf, lengths
        if self.mode == "stochastic" and (V % 8 != 0 or p.data_ptr() % 16 or (q is not None and q.data_ptr() % 16)):
            # the TMA sampler needs 32-byte rows (V % 8 == 0) and 16-byte aligned p / q (persist_eligible,
            # csrc/stream.cu): the stage-by-stage kernels serve any V and alignment
            self._check(lib.tetris_select_f64(sel_conf.data_ptr(), _ptr(sel_len), self.Bg, k, self.C, 0,
                                              self.windows_all.data_ptr(), self.win_offsets.data_ptr(), None,
                                              self.stats.data_ptr(), self.status.data_ptr(), ws.ptr, ws.nbytes, s))
            if events is not None:
                events[1].record()
            packed = self.u_layout == "packed"
            self._check(lib.tetris_verify_stochastic_f32(
                p.data_ptr(), q.data_ptr(), _ptr(d), self.windows.data_ptr(),
                self.win_offsets.data_ptr() if packed else None, _ptr(u_acc), u_res.data_ptr(), B, k, V,
                self.accepted.data_ptr(), self.out_tok.data_ptr(), self.mass.data_ptr(), self.status.data_ptr(),
                ws.ptr, ws.nbytes, s))
            if events is not None:
                events[2].record()
            self._check(lib.tetris_compact(self.accepted.data_ptr(), self.out_tok.data_ptr(), _ptr(d), _ptr(cap), B,
                                           k, self.offsets.data_ptr(), self.tokens.data_ptr(), s))
            if events is not None:
                events[3].record()
            return
        if self.mode == "stochastic" and self.fused:
            # small batch: the whole step is ONE launch (tetris_step_stochastic_f32 -> the sampler with the selection
            # as its prologue, csrc/stream.cu fused_select); events bracket [nothing | the step | nothing]
            if events is not None:
                events[1].record()
            self._check(lib.tetris_step_stochastic_f32(
                sel_conf.data_ptr(), _ptr(sel_len), self.Bg, k, self.C, self.rank * B, B, p.data_ptr(), q.data_ptr(),
                d.data_ptr(), u_acc.data_ptr(), 0, u_res.data_ptr(), _ptr(cap), V, self.windows_all.data_ptr(),
                self.win_offsets.data_ptr(), self.accepted.data_ptr(), self.out_tok.data_ptr(), self.mass.data_ptr(),
                self.offsets.data_ptr(), self.tokens.data_ptr(), self.stats.data_ptr(), self.status.data_ptr(),
                ws.ptr, ws.nbytes, s))
            if events is not None:
                events[2].record()
                events[3].record()
            return
        if self.mode == "stochastic":
            # == tetris_step_stochastic_f32, called as its two halves so an event can sit between the kernels
            rc = lib.tetris_select_accept_f32(
                sel_conf.data_ptr(), _ptr(sel_len), self.Bg, k, self.C, self.rank * B, B, p.data_ptr(), q.data_ptr(),
                d.data_ptr(), u_acc.data_ptr(), int(self.u_layout == "packed"), _ptr(cap), V,
                self.windows_all.data_ptr(), self.win_offsets.data_ptr(), self.accepted.data_ptr(),
                self.offsets.data_ptr(), self.tokens.data_ptr(), self.stats.data_ptr(), self.status.data_ptr(),
                ws.ptr, ws.nbytes, s)
            self._check(rc)
            if events is not None:
                events[1].record()
            if self.uses_spec:
                # the speculative sampler: rows that do not depend on the selection stream while it runs
                len_local = None if sel_len is None else sel_len[self.rank * B:(self.rank + 1) * B]
                rc = lib.tetris_resample_spec_f32(
                    p.data_ptr(), q.data_ptr(), u_res.data_ptr(), u_acc.data_ptr(), _ptr(len_local), B, k, V,
                    d.data_ptr(), self.accepted.data_ptr(), self.offsets.data_ptr(), self.out_tok.data_ptr(),
                    self.mass.data_ptr(), self.tokens.data_ptr(), self.status.data_ptr(), ws.ptr, ws.nbytes, s)
            else:
                rc = lib.tetris_resample_f32(p.data_ptr(), q.data_ptr(), u_res.data_ptr(), B, k, V, d.data_ptr(),
                                             self.accepted.data_ptr(), self.offsets.data_ptr(),
                                             self.out_tok.data_ptr(), self.mass.data_ptr(), self.tokens.data_ptr(),
                                             self.status.data_ptr(), ws.ptr, ws.nbytes, s)
            self._check(rc)
            if events is not None:
                events[2].record()
                events[3].record()
            return
        if events is not None:
            # stage timing (eager): the same results stage by stage, so an event can sit between the selection and
            # the argmax stream (the product path below fuses the row list into the selector's epilogue)
            self._check(lib.tetris_select_f64(sel_conf.data_ptr(), _ptr(sel_len), self.Bg, k, self.C, 0,
                                              self.windows_all.data_ptr(), self.win_offsets.data_ptr(), None,
                                              self.stats.data_ptr(), self.status.data_ptr(), ws.ptr, ws.nbytes, s))
            events[1].record()
            self._check(lib.tetris_verify_greedy_compact_f32(
                p.data_ptr(), d.data_ptr(), self.windows.data_ptr(), _ptr(cap), B, k, V, self.accepted.data_ptr(),
                self.out_tok.data_ptr(), self.offsets.data_ptr(), self.tokens.data_ptr(), self.status.data_ptr(),
                ws.ptr, ws.nbytes, s))
            events[2].record()
            events[3].record()
            return
        # == tetris_step_greedy_f32 (select1 with the row-list epilogue, then the persistent argmax stream with the
        # verdicts and the compaction)
        rc = lib.tetris_step_greedy_f32(
            sel_conf.data_ptr(), _ptr(sel_len), self.Bg, k, self.C, self.rank * B, B, p.data_ptr(), d.data_ptr(),
            _ptr(cap), V, self.windows_all.data_ptr(), self.win_offsets.data_ptr(), self.accepted.data_ptr(),
            self.out_tok.data_ptr(), self.offsets.data_ptr(), self.tokens.data_ptr(), self.stats.data_ptr(),
            self.status.data_ptr(), ws.ptr, ws.nbytes, s)
        self._check(rc)

    def _dist_native(self, p, q) -> bool:
        """The native sharded step serves the dense-uniform TETRIS step; the stochastic form needs the TMA sampler's
        V % 8 == 0 and 16-byte aligned p / q (the greedy step falls back inside the library)."""
        if self.u_layout != "dense" or self.policy != "tetris":
            return False
        return self.mode == "greedy" or (self.V % 8 == 0 and p.data_ptr() % 16 == 0 and q.data_ptr() % 16 == 0)

    def _run_dist(self, conf, lengths, p, q, d, u_acc, u_res, cap) -> None:
        """Request-sharded step over NCCL in one library call: the score all-gather (one NCCL group on the current
        stream), the global selection over the gathered rows, this rank's verification and compaction."""
        lib, ws, s = self._lib, self.ws, torch.cuda.current_stream().cuda_stream
        B, k, V = self.B, self.k, self.V
        len_all = None if lengths is None else self.len_all
        if self.mode == "stochastic":
            rc = lib.tetris_dist_step_stochastic_f32(
                conf.data_ptr(), _ptr(lengths), B, k, self.C, p.data_ptr(), q.data_ptr(), d.data_ptr(),
                u_acc.data_ptr(), u_res.data_ptr(), _ptr(cap), V, self._comm, self.conf_all.data_ptr(), _ptr(len_all),
                self.windows_all.data_ptr(), self.win_offsets.data_ptr(), self.accepted.data_ptr(),
                self.out_tok.data_ptr(), self.mass.data_ptr(), self.offsets.data_ptr(), self.tokens.data_ptr(),
                self.stats.data_ptr(), self.status.data_ptr(), ws.ptr, ws.nbytes, s)
        else:
            rc = lib.tetris_dist_step_greedy_f32(
                conf.data_ptr(), _ptr(lengths), B, k, self.C, p.data_ptr(), _ptr(d), _ptr(cap), V, self._comm,
                self.conf_all.data_ptr(), _ptr(len_all), self.windows_all.data_ptr(), self.win_offsets.data_ptr(),
                self.accepted.data_ptr(), self.out_tok.data_ptr(), self.offsets.data_ptr(), self.tokens.data_ptr(),
                self.stats.data_ptr(), self.status.data_ptr(), ws.ptr, ws.nbytes, s)
        self._check(rc)

    def run_logits(self, conf, lengths, zp, lse_p, zq, lse_q, d, u_acc, u_res, cap=None, events=None) -> None:
        """The stochastic step on LOGITS: zp [B, k+1, V] / zq [B, k, V] bf16 logits with their row
        log-sum-exp lse_p [B, k+1] / lse_q [B, k] f32 (the LM head's softmax normaliser); every probability is the
        logits contract's prob(z, lse) (include/tetris_b200.h), computed inside the kernels.  Results equal run() on
        p = probs_from_logits(zp, lse_p), q = probs_from_logits(zq, lse_q); half the streamed bytes.  Same launches
        as run() (select + accept, then the persistent sampler); events bracket [select | sampler | nothing]."""
        if self.mode != "stochastic" or self.policy != "tetris":
            raise ValueError("run_logits is the stochastic TETRIS step")
        B, k, V = self.B, self.k, self.V
        for name, t, shape in (("zp", zp, (B, k + 1, V)), ("zq", zq, (B, k, V))):
            if t.dtype != torch.bfloat16 or tuple(t.shape) != shape or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous bfloat16 tensor of shape {shape}")
        for name, t, shape in (("lse_p", lse_p, (B, k + 1)), ("lse_q", lse_q, (B, k))):
            if t.dtype != _F32 or tuple(t.shape) != shape or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float32 tensor of shape {shape}")
        if V % 8 or zp.data_ptr() % 16 or zq.data_ptr() % 16:
            raise ValueError("the logits step needs V % 8 == 0 and 16-byte aligned logits")
        lib, ws, s = self._lib, self.ws, torch.cuda.current_stream().cuda_stream
        if events is not None:
            events[0].record()
        if self._comm is not None and events is None and self.u_layout == "dense":
            len_all = None if lengths is None else self.len_all
            self._check(lib.tetris_dist_step_stochastic_bf16(
                conf.data_ptr(), _ptr(lengths), B, k, self.C, zp.data_ptr(), lse_p.data_ptr(), zq.data_ptr(),
                lse_q.data_ptr(), d.data_ptr(), u_acc.data_ptr(), u_res.data_ptr(), _ptr(cap), V, self._comm,
                self.conf_all.data_ptr(), _ptr(len_all), self.windows_all.data_ptr(), self.win_offsets.data_ptr(),
                self.accepted.data_ptr(), self.out_tok.data_ptr(), self.mass.data_ptr(), self.offsets.data_ptr(),
                self.tokens.data_ptr(), self.stats.data_ptr(), self.status.data_ptr(), ws.ptr, ws.nbytes, s))
            return
        if self.world > 1 and self.group is not None:
            from .dist import gather_scores

            gather_scores(self.conf_all, self.len_all, conf, lengths, self.group)
            sel_conf, sel_len = self.conf_all, self.len_all
        else:
            sel_conf, sel_len = conf, lengths
        if self.fused:
            if events is not None:
                events[1].record()
            self._check(lib.tetris_step_stochastic_bf16(
                sel_conf.data_ptr(), _ptr(sel_len), self.Bg, k, self.C, self.rank * B, B, zp.data_ptr(),
                lse_p.data_ptr(), zq.data_ptr(), lse_q.data_ptr(), d.data_ptr(), u_acc.data_ptr(), 0,
                u_res.data_ptr(), _ptr(cap), V, self.windows_all.data_ptr(), self.win_offsets.data_ptr(),
                self.accepted.data_ptr(), self.out_tok.data_ptr(), self.mass.data_ptr(), self.offsets.data_ptr(),
                self.tokens.data_ptr(), self.stats.data_ptr(), self.status.data_ptr(), ws.ptr, ws.nbytes, s))
            if events is not None:
                events[2].record()
                events[3].record()
            return
        self._check(lib.tetris_select_accept_bf16(
            sel_conf.data_ptr(), _ptr(sel_len), self.Bg, k, self.C, self.rank * B, B, zp.data_ptr(),
            lse_p.data_ptr(), zq.data_ptr(), lse_q.data_ptr(), d.data_ptr(), u_acc.data_ptr(),
            int(self.u_layout == "packed"), _ptr(cap), V, self.windows_all.data_ptr(), self.win_offsets.data_ptr(),
            self.accepted.data_ptr(), self.offsets.data_ptr(), self.tokens.data_ptr(), self.stats.data_ptr(),
            self.status.data_ptr(), ws.ptr, ws.nbytes, s))
        if events is not None:
            events[1].record()
        spec = self.uses_spec
        len_local = None if (sel_len is None or not spec) else sel_len[self.rank * B:(self.rank + 1) * B]
        self._check(lib.tetris_resample_bf16(
            zp.data_ptr(), lse_p.data_ptr(), zq.data_ptr(), lse_q.data_ptr(), u_res.data_ptr(),
            u_acc.data_ptr() if spec else None, _ptr(len_local), B, k, V, d.data_ptr(), self.accepted.data_ptr(),
            self.offsets.data_ptr(), self.out_tok.data_ptr(), self.mass.data_ptr(), self.tokens.data_ptr(),
            self.status.data_ptr(), ws.ptr, ws.nbytes, s))
        if events is not None:
            events[2].record()
            events[3].record()

    def _run_fixed(self, lengths, p, q, d, u_acc, u_res, cap, events, window) -> None:
        """Baseline step (fixed window / sd / dsd common window, clamped to each depth): windows kernel, then the same
        verification and compaction kernels as the TETRIS step, so step times compare apples to apples."""
        lib, ws, s = self._lib, self.ws, torch.cuda.current_stream().cuda_stream
        B, k, V = self.B, self.k, self.V
        w = self.C // B if window is None else int(window)
        self._check(lib.tetris_uniform_windows(_ptr(lengths), B, k, w, self.windows.data_ptr(),
                                               self.win_offsets.data_ptr(), s))
        if events is not None:
            events[1].record()
        if self.mode == "stochastic":
            self._check(lib.tetris_verify_stochastic_f32(
                p.data_ptr(), q.data_ptr(), d.data_ptr(), self.windows.data_ptr(),
                self.win_offsets.data_ptr() if self.u_layout == "packed" else None, u_acc.data_ptr(),
                u_res.data_ptr(), B, k, V, self.accepted.data_ptr(), self.out_tok.data_ptr(), self.mass.data_ptr(),
                self.status.data_ptr(), ws.ptr, ws.nbytes, s))
        else:
            self._check(lib.tetris_verify_greedy_compact_f32(
                p.data_ptr(), d.data_ptr(), self.windows.data_ptr(), _ptr(cap), B, k, V, self.accepted.data_ptr(),
                self.out_tok.data_ptr(), self.offsets.data_ptr(), self.tokens.data_ptr(), self.status.data_ptr(),
                ws.ptr, ws.nbytes, s))
            if events is not None:
                events[2].record()
                events[3].record()
            return
        if events is not None:
            events[2].record()
        self._check(lib.tetris_compact(self.accepted.data_ptr(), self.out_tok.data_ptr(), d.data_ptr(), _ptr(cap), B,
                                       k, self.offsets.data_ptr(), self.tokens.data_ptr(), s))
        if events is not None:
            events[3].record()

    def _check(self, rc: int) -> None:
        if rc != N.OK:
            msg = self._lib.tetris_last_error().decode(errors="replace")
            raise ValueError(msg) if rc == N.INVALID_ARGUMENT else N.TetrisError(rc, msg)

    @property
    def fused(self) -> bool:
        """True when the stochastic step is ONE launch: the selection runs as the sampler's prologue (small batches,
        Bg * k <= FUSED_MAX_CELLS, dense uniforms; csrc/stream.cu fused_select)."""
        return (self.mode == "stochastic" and self.policy == "tetris" and self.u_layout == "dense"
                and self.Bg * self.k <= FUSED_MAX_CELLS and self.Bg <= FUSED_MAX_ROWS and not _NO_FUSED)

    @property
    def uses_spec(self) -> bool:
        """True when the stochastic step runs the speculative sampler (tetris_resample_spec_f32)."""
        return (self.mode == "stochastic" and self.policy == "tetris" and self.u_layout == "dense"
                and self.B <= self.spec_max and self.B * -(-self.V // 8192) >= SPEC_MIN_CHUNKS and not _NO_SPEC)

    @property
    def launches_per_step(self) -> int:
        # stochastic: select kernel (+ accept CTAs), persist_stream_kernel (streaming + descent + token stream);
        # greedy: select1_kernel (+ row list), persist_greedy_kernel (argmax stream + verdicts + compaction), plus
        # greedy_rowmap_kernel when the batch is too large for the single-CTA selector (B * k > 16384);
        # fixed-window baseline: windows, accept, stream, compact (stochastic) or windows, rowmap, greedy stream
        # (V % 8 == 0 and 16-byte aligned p; otherwise the greedy fallback adds its compact launch)
        if self.policy == "fixed":
            return 4 if self.mode == "stochastic" else 3
        if self.mode == "stochastic":
            if self.V % 8 != 0:
                return 3  # select, verify (one sample_kernel), compact
            return 1 if self.fused else 2
        if self.Bg * self.k <= FUSED_MAX_CELLS and self.Bg <= FUSED_MAX_ROWS and self.V % 8 == 0 and not _NO_FUSED:
            return 1  # the one-launch greedy step (selection as the argmax stream's prologue)
        return 2 if self.Bg * self.k <= 16384 and self.Bg <= 4096 else 3


class _MappedTensor:
    """Stand-in exposing a device address for a pinned host tensor (zero-copy reads by the kernels).  Memory that the
    library had to register (pageable input) is unregistered when this object goes away."""

    def __init__(self, host: torch.Tensor):
        if host.is_cuda or not host.is_contiguous():
            raise ValueError("expected a contiguous host tensor")
        self.host = host
        self._ptr = host.data_ptr()
        self._dev = N.map_host(self._ptr, host.numel() * host.element_size())

    def data_ptr(self) -> int:
        return self._dev

    def __del__(self):
        try:
            N.unmap_host(self._ptr)
        except Exception:
            pass


class HostTetrisStep:
    """The same step for HOST-resident inputs (the end-to-end API): small per-request inputs (conf, lengths, draft
    tokens, uniforms) are copied host->device; the large target/draft probability tensors stay in pinned host memory
    and only the rows the step needs cross the host link; the compacted token stream and per-request results are
    copied back into pinned host buffers.  `run` is stream-ordered; call `torch.cuda.current_stream().synchronize()`
    (or `wait()`) before reading `tokens_host`."""

    def __init__(self, B: int, k: int, V: int, capacity: int, p_host: torch.Tensor, q_host: Optional[torch.Tensor],
                 mode: str = "stochastic", device="cuda", transfer: str = "staged"):
        """transfer: "staged" (after the selection a gather kernel copies the needed rows host->device over the
        mapping -- tetris_step_stochastic_staged_f32: the residual / bonus row of each request into a [2B, V] staging
        buffer; tetris_step_greedy_staged_f32: rows 0..w_b of each request into their place of a [B, k+1, V] device
        copy) or "zero-copy" (the streaming kernels read the rows from pinned host memory themselves).  Neither waits
        on the host.  q_host may be None (or empty) when k == 0 or mode == "greedy"."""
        if transfer not in ("staged", "zero-copy"):
            raise ValueError(f"transfer must be 'staged' or 'zero-copy', got {transfer!r}")
        self.step = TetrisStep(B, k, V, capacity, mode=mode, device=device)
        dev = self.step.device
        self.mode = mode
        # the staged paths copy 16-byte words and the stochastic one feeds the TMA sampler (32-byte rows): other
        # vocabulary sizes and misaligned views read through the mapping
        aligned = p_host.data_ptr() % 16 == 0 and (q_host is None or q_host.numel() == 0 or q_host.data_ptr() % 16 == 0)
        self.transfer = transfer if aligned and V % (4 if mode == "greedy" else 8) == 0 else "zero-copy"
        if q_host is not None and q_host.numel() == 0:
            q_host = None
        if mode == "stochastic" and k > 0 and q_host is None:
            raise ValueError("q_host is required for stochastic verification with k > 0")
        self.p_host, self.q_host = p_host, q_host
        self.p = _MappedTensor(p_host)
        # k == 0 (nothing drafted): no draft rows exist; an empty device tensor stands in (null pointer in the ABI)
        self.q = _MappedTensor(q_host) if q_host is not None else torch.empty(B, 0, V, dtype=_F32, device=dev)
        if self.transfer == "staged" and mode == "stochastic":
            self.staging = torch.empty(2 * B, V, dtype=torch.float32, device=dev)
        elif self.transfer == "staged":
            self.p_dev = torch.empty(B, k + 1, V, dtype=torch.float32, device=dev)
        self.conf = torch.empty(B, k, dtype=_F64, device=dev)
        self.lengths = torch.empty(B, dtype=_I32, device=dev)
        self.d = torch.empty(B, k, dtype=_I32, device=dev)
        self.u_acc = torch.empty(B, k, dtype=_F64, device=dev)
        self.u_res = torch.empty(B, dtype=_F64, device=dev)
        self.offsets_host = torch.empty(B + 1, dtype=_I32).pin_memory()
        self.tokens_host = torch.empty(B * (k + 1), dtype=_I32).pin_memory()
        self.accepted_host = torch.empty(B, dtype=_I32).pin_memory()
        self.B, self.k, self.V = B, k, V

    def h2d_bytes(self) -> int:
        """Bytes of the explicit per-request input copies (the probability rows come on top, see the bench)."""
        B, k = self.B, self.k
        n = B * k * 8 + B * 4 + B * k * 4
        return n + (B * k * 8 + B * 8 if self.mode == "stochastic" else 0)

    def d2h_bytes(self) -> int:
        return (self.B + 1) * 4 + self.B * (self.k + 1) * 4 + self.B * 4

    def run(self, conf_h, lengths_h, d_h, u_acc_h=None, u_res_h=None) -> None:
        self.conf.copy_(conf_h, non_blocking=True)
        self.lengths.copy_(lengths_h, non_blocking=True)
        self.d.copy_(d_h, non_blocking=True)
        if u_acc_h is not None:
            self.u_acc.copy_(u_acc_h, non_blocking=True)
            self.u_res.copy_(u_res_h, non_blocking=True)
        st = self.step
        s = torch.cuda.current_stream().cuda_stream
        if self.transfer == "staged" and st.group is None and self.mode == "stochastic":
            st._check(st._lib.tetris_step_stochastic_staged_f32(
                self.conf.data_ptr(), self.lengths.data_ptr(), self.B, self.k, st.C, self.p_host.data_ptr(),
                _ptr(self.q_host), self.d.data_ptr(), self.u_acc.data_ptr(), self.u_res.data_ptr(), None,
                self.V, self.staging.data_ptr(), st.windows_all.data_ptr(),
                st.win_offsets.data_ptr(), st.accepted.data_ptr(), st.out_tok.data_ptr(), st.mass.data_ptr(),
                st.offsets.data_ptr(), st.tokens.data_ptr(), st.stats.data_ptr(), st.status.data_ptr(), st.ws.ptr,
                st.ws.nbytes, s))
        elif self.transfer == "staged" and st.group is None:
            st._check(st._lib.tetris_step_greedy_staged_f32(
                self.conf.data_ptr(), self.lengths.data_ptr(), self.B, self.k, st.C, self.p_host.data_ptr(),
                self.d.data_ptr(), None, self.V, self.p_dev.data_ptr(), st.windows_all.data_ptr(), st.win_offsets.data_ptr(), st.accepted.data_ptr(), st.out_tok.data_ptr(),
                st.offsets.data_ptr(), st.tokens.data_ptr(), st.stats.data_ptr(), st.status.data_ptr(), st.ws.ptr,
                st.ws.nbytes, s))
        else:
            st.run(self.conf, self.lengths, self.p, self.q, self.d, self.u_acc, self.u_res)
        self.offsets_host.copy_(st.offsets, non_blocking=True)
        self.tokens_host.copy_(st.tokens, non_blocking=True)
        self.accepted_host.copy_(st.accepted, non_blocking=True)


class HostLogitStep:
    """HostTetrisStep for LOGITS: zp_host [B, k+1, V] / zq_host [B, k, V] bf16 and lse_p_host [B, k+1] / lse_q_host
    [B, k] f32 in pinned host memory (tetris_step_stochastic_staged_bf16: after the selection a gather kernel copies
    the needed bf16 rows host->device -- half the host-link bytes of the fp32 form)."""

    def __init__(self, B: int, k: int, V: int, capacity: int, zp_host: torch.Tensor, lse_p_host: torch.Tensor,
                 zq_host: torch.Tensor, lse_q_host: torch.Tensor, device="cuda"):
        for name, t in (("zp_host", zp_host), ("zq_host", zq_host), ("lse_p_host", lse_p_host),
                        ("lse_q_host", lse_q_host)):
            if t.is_cuda or not t.is_contiguous() or not t.is_pinned():
                raise ValueError(f"{name} must be a contiguous pinned host tensor")
        if zp_host.dtype != torch.bfloat16 or zq_host.dtype != torch.bfloat16:
            raise ValueError("zp_host / zq_host must be bfloat16")
        if V % 8:
            raise ValueError("the logits step needs V % 8 == 0")
        self.step = TetrisStep(B, k, V, capacity, mode="stochastic", device=device)
        dev = self.step.device
        self.host = (zp_host, lse_p_host, zq_host, lse_q_host)
        self.staging = torch.empty(2 * B, V, dtype=torch.bfloat16, device=dev)
        self.lse_staging = torch.empty(2 * B, dtype=_F32, device=dev)
        self.conf = torch.empty(B, k, dtype=_F64, device=dev)
        self.lengths = torch.empty(B, dtype=_I32, device=dev)
        self.d = torch.empty(B, k, dtype=_I32, device=dev)
        self.u_acc = torch.empty(B, k, dtype=_F64, device=dev)
        self.u_res = torch.empty(B, dtype=_F64, device=dev)
        self.offsets_host = torch.empty(B + 1, dtype=_I32).pin_memory()
        self.tokens_host = torch.empty(B * (k + 1), dtype=_I32).pin_memory()
        self.accepted_host = torch.empty(B, dtype=_I32).pin_memory()
        self.B, self.k, self.V = B, k, V

    def h2d_bytes(self) -> int:
        B, k = self.B, self.k
        return B * k * 8 + B * 4 + B * k * 4 + B * k * 8 + B * 8

    def d2h_bytes(self) -> int:
        return (self.B + 1) * 4 + self.B * (self.k + 1) * 4 + self.B * 4

    def run(self, conf_h, lengths_h, d_h, u_acc_h, u_res_h) -> None:
        for dst, src in ((self.conf, conf_h), (self.lengths, lengths_h), (self.d, d_h), (self.u_acc, u_acc_h),
                         (self.u_res, u_res_h)):
            dst.copy_(src, non_blocking=True)
        st = self.step
        zp, lp, zq, lq = self.host
        st._check(st._lib.tetris_step_stochastic_staged_bf16(
            self.conf.data_ptr(), self.lengths.data_ptr(), self.B, self.k, st.C, zp.data_ptr(), lp.data_ptr(),
            zq.data_ptr(), lq.data_ptr(), self.d.data_ptr(), self.u_acc.data_ptr(), self.u_res.data_ptr(), None,
            self.V, self.staging.data_ptr(), self.lse_staging.data_ptr(), st.windows_all.data_ptr(), st.win_offsets.data_ptr(), st.accepted.data_ptr(),
            st.out_tok.data_ptr(), st.mass.data_ptr(), st.offsets.data_ptr(), st.tokens.data_ptr(),
            st.stats.data_ptr(), st.status.data_ptr(), st.ws.ptr, st.ws.nbytes, torch.cuda.current_stream().cuda_stream))
        self.offsets_host.copy_(st.offsets, non_blocking=True)
        self.tokens_host.copy_(st.tokens, non_blocking=True)
        self.accepted_host.copy_(st.accepted, non_blocking=True)
