"""ctypes wrapper of the CPU oracle (oracle/tetris_oracle.c).  TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs, as the checker.  Every
function takes and returns numpy arrays; see tetris_oracle.c for the reference file:line each one restates.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_build" / "libtetris_oracle.so"
_lib = None

_p = C.c_void_p


def _load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            import sys

            sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
            from paper_2502_15197_b200._build import build_oracle

            build_oracle()
        lib = C.CDLL(str(LIB_PATH))
        lib.oracle_select.restype = C.c_int
        lib.oracle_select.argtypes = [_p, _p, C.c_int, C.c_int, C.c_int64, C.c_int, _p, _p, _p]
        lib.oracle_expected_accepted.restype = C.c_double
        lib.oracle_expected_accepted.argtypes = [_p, _p, _p, C.c_int, C.c_int]
        lib.oracle_verify_token.restype = C.c_int
        lib.oracle_verify_token.argtypes = [C.c_double, C.c_double, C.c_double]
        lib.oracle_verify_matrix.restype = None
        lib.oracle_verify_matrix.argtypes = [_p, _p, _p, _p, C.c_int, C.c_int, _p]
        lib.oracle_sample_f64.restype = C.c_int
        lib.oracle_sample_f64.argtypes = [_p, _p, C.c_int, C.c_double, _p]
        lib.oracle_sample_f32.restype = C.c_int
        lib.oracle_sample_f32.argtypes = [_p, _p, C.c_int, C.c_double, _p]
        lib.oracle_residual_f64.restype = C.c_int
        lib.oracle_residual_f64.argtypes = [_p, _p, C.c_int, _p, _p]
        lib.oracle_verify_stochastic_f32.restype = None
        lib.oracle_verify_stochastic_f32.argtypes = [_p, _p, _p, _p, _p, _p, _p, C.c_int, C.c_int, C.c_int, _p, _p,
                                                     _p, C.c_int]
        lib.oracle_verify_greedy_f32.restype = None
        lib.oracle_verify_greedy_f32.argtypes = [_p, _p, _p, C.c_int, C.c_int, C.c_int, _p, _p, C.c_int]
        lib.oracle_probs_from_logits_bf16.restype = None
        lib.oracle_probs_from_logits_bf16.argtypes = [_p, _p, C.c_int64, C.c_int, _p]
        lib.oracle_compact.restype = None
        lib.oracle_compact.argtypes = [_p, _p, _p, _p, C.c_int, C.c_int, _p, _p]
        _lib = lib
    return _lib


def _a(x, dtype):
    return np.ascontiguousarray(x, dtype=dtype)


def _ptr(a):
    return None if a is None else a.ctypes.data


def select(vals, capacity, lengths=None, vals_are_cum=False):
    """heapq port of select_tetris(cumulative_products(...)) -> (windows i32[B], cum f64[B,k], stats i64[4])."""
    vals = _a(vals, np.float64)
    B, k = vals.shape
    ln = None if lengths is None else _a(lengths, np.int32)
    windows = np.zeros(B, np.int32)
    cum = np.zeros((B, k), np.float64)
    stats = np.zeros(4, np.int64)
    rc = _load().oracle_select(_ptr(vals), _ptr(ln), B, k, int(capacity), int(vals_are_cum), _ptr(windows),
                               _ptr(cum), _ptr(stats))
    if rc:
        raise ValueError(f"capacity must be >= 0, got {capacity}")
    return windows, cum, stats


def expected_accepted(alpha, windows, lengths=None):
    alpha = _a(alpha, np.float64)
    B, k = alpha.shape
    w = _a(windows, np.int32)
    return float(_load().oracle_expected_accepted(_ptr(alpha), None, _ptr(w), B, k))


def verify_token(p_draft, p_target, token, u) -> bool:
    """verify_token (accept_model.py:291-313) on fp64 rows."""
    return bool(_load().oracle_verify_token(float(p_draft[token]), float(p_target[token]), float(u)))


def verify_matrix(alpha, windows, u):
    alpha = _a(alpha, np.float64)
    B, k = alpha.shape
    w = _a(windows, np.int32)
    off = np.zeros(B, np.int32)
    off[1:] = np.cumsum(w)[:-1]
    u = _a(u, np.float64)
    acc = np.zeros(B, np.int32)
    _load().oracle_verify_matrix(_ptr(alpha), _ptr(w), _ptr(off), _ptr(u), B, k, _ptr(acc))
    return acc


def sample(p, u, q=None):
    """Sampling contract on one row: weights max(0, p - q) or max(0, p).  Returns (index, mass)."""
    p = np.ascontiguousarray(p)
    if p.dtype == np.float32:
        fn, q = _load().oracle_sample_f32, (None if q is None else _a(q, np.float32))
    else:
        p = _a(p, np.float64)
        fn, q = _load().oracle_sample_f64, (None if q is None else _a(q, np.float64))
    mass = C.c_double(0.0)
    idx = fn(_ptr(p), _ptr(q), p.shape[0], float(u), C.addressof(mass))
    return int(idx), float(mass.value)


def residual(p_draft, p_target):
    ps = _a(p_draft, np.float64)
    pt = _a(p_target, np.float64)
    out = np.zeros_like(ps)
    mass = C.c_double(0.0)
    rc = _load().oracle_residual_f64(_ptr(ps), _ptr(pt), ps.shape[0], _ptr(out), C.addressof(mass))
    return out, float(mass.value), rc


def verify_stochastic(p, q, d, windows, u_acc, u_res, win_offsets=None, nthreads=1):
    p = _a(p, np.float32)
    q = _a(q, np.float32)
    B, k1, V = p.shape
    k = k1 - 1
    d = _a(d, np.int32)
    w = _a(windows, np.int32)
    woff = None if win_offsets is None else _a(win_offsets, np.int32)
    u_acc = _a(u_acc, np.float64)
    u_res = _a(u_res, np.float64)
    acc = np.zeros(B, np.int32)
    tok = np.zeros(B, np.int32)
    mass = np.zeros(B, np.float64)
    _load().oracle_verify_stochastic_f32(_ptr(p), _ptr(q), _ptr(d), _ptr(w), _ptr(woff), _ptr(u_acc), _ptr(u_res), B,
                                         k, V, _ptr(acc), _ptr(tok), _ptr(mass), int(nthreads))
    return acc, tok, mass


def verify_greedy(p, d, windows, nthreads=1):
    p = _a(p, np.float32)
    B, k1, V = p.shape
    d = _a(d, np.int32)
    w = _a(windows, np.int32)
    acc = np.zeros(B, np.int32)
    tok = np.zeros(B, np.int32)
    _load().oracle_verify_greedy_f32(_ptr(p), _ptr(d), _ptr(w), B, k1 - 1, V, _ptr(acc), _ptr(tok), int(nthreads))
    return acc, tok


def compact(accepted, out_tok, d, cap=None):
    acc = _a(accepted, np.int32)
    tok = _a(out_tok, np.int32)
    d = _a(d, np.int32)
    B, k = d.shape
    capa = None if cap is None else _a(cap, np.int32)
    offsets = np.zeros(B + 1, np.int32)
    tokens = np.zeros(B * (k + 1), np.int32)
    _load().oracle_compact(_ptr(acc), _ptr(tok), _ptr(d), _ptr(capa), B, k, _ptr(offsets), _ptr(tokens))
    return offsets, tokens[: offsets[-1]]


def probs_from_logits_bf16(z_bits, lse):
    """The logits contract (include/tetris_b200.h): z_bits [..., V] uint16 bf16 bits, lse [...] f32 -> fp32 probs."""
    z = _a(z_bits, np.uint16)
    lse = _a(lse, np.float32)
    V = z.shape[-1]
    R = int(np.prod(z.shape[:-1]))
    assert lse.size == R
    out = np.empty(z.shape, np.float32)
    _load().oracle_probs_from_logits_bf16(_ptr(z), _ptr(lse), R, V, _ptr(out))
    return out
