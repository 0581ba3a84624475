"""ctypes binding of libtetris_b200.so (the C ABI declared in include/tetris_b200.h).

There is no fallback: if the shared library is missing or fails to load, every op raises NativeLibraryError.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_native" / "libtetris_b200.so"
if os.environ.get("TETRIS_LIB_VARIANT"):  # A/B experiments: another build of the same ABI under _native/
    LIB_PATH = LIB_PATH.parent / os.environ["TETRIS_LIB_VARIANT"]

OK = 0
INVALID_ARGUMENT = 1
DEGENERATE_RESIDUAL = 2
CUDA_ERROR = 3
NCCL_ERROR = 4

ST_BAD_VALUE = 1
ST_DEGENERATE = 2
ST_BAD_TOKEN = 4
ST_BAD_UNIFORM = 8
ST_BAD_WINDOW = 16
ST_STREAM_EXHAUSTED = 32

OP_SELECT = 1
OP_VERIFY = 2
OP_ALL = 3

# contract constants (must equal the header's; checked in tests/test_abi.py)
LANE_ELEMS = 8
SEG_ELEMS = 256
WARP_SEGS = 4
CHUNK_WARPS = 8
CHUNK_ELEMS = 8192
MAX_K = 255


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or failed to load; there is deliberately no CPU fallback."""


class TetrisError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_sz = C.c_size_t

_SIGNATURES = {
    "tetris_last_error": (C.c_char_p, []),
    "tetris_abi_version": (C.c_int, []),
    "tetris_debug_timestamps": (C.c_int, [_p]),
    "tetris_map_host": (C.c_int, [_p, _sz, C.POINTER(C.c_void_p)]),
    "tetris_unmap_host": (C.c_int, [_p]),
    "tetris_spec_max_requests": (C.c_int, []),
    "tetris_workspace_bytes": (_sz, [C.c_int, _i32, _i32, _i32]),
    "tetris_workspace_init": (C.c_int, [_p, _sz, _p]),
    "tetris_select_f64": (C.c_int, [_p, _p, _i32, _i32, _i64, _i32, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_heap_stats_f64": (C.c_int, [_p, _p, _i32, _i32, _i64, _p, _p, _sz, _p]),
    "tetris_expected_accepted_f64": (C.c_int, [_p, _p, _p, _i32, _i32, _p, _p, _p]),
    "tetris_verify_matrix_f64": (C.c_int, [_p, _p, _p, _p, _p, _i32, _i32, _p, _p, _p]),
    "tetris_verify_tokens_f64": (C.c_int, [_p, _p, _p, _p, _i32, _i32, _p, _p, _p]),
    "tetris_verify_stochastic_f32": (
        C.c_int, [_p, _p, _p, _p, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_select_accept_f32": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _i32, _i32, _p, _p, _p, _p, _i32, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p,
                  _sz, _p]),
    "tetris_resample_f32": (C.c_int, [_p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_resample_spec_f32": (
        C.c_int, [_p, _p, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_step_stochastic_f32": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _i32, _i32, _p, _p, _p, _p, _i32, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p,
                  _p, _p, _p, _sz, _p]),
    "tetris_step_stochastic_bf16": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _i32, _i32, _p, _p, _p, _p, _p, _p, _i32, _p, _p, _i32, _p, _p, _p, _p, _p,
                  _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_select_accept_bf16": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _i32, _i32, _p, _p, _p, _p, _p, _p, _i32, _p, _i32, _p, _p, _p, _p, _p, _p,
                  _p, _p, _sz, _p]),
    "tetris_resample_bf16": (
        C.c_int, [_p, _p, _p, _p, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_probs_from_logits_bf16": (C.c_int, [_p, _p, _i64, _i32, _p, _p]),
    "tetris_verify_greedy_f32": (C.c_int, [_p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p, _sz, _p]),
    "tetris_step_stochastic_staged_f32": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _p, _p, _p, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                  _sz, _p]),
    "tetris_step_stochastic_staged_bf16": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                  _p, _p, _p, _sz, _p]),
    "tetris_step_greedy_staged_f32": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_step_greedy_f32": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _i32, _i32, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _sz,
                  _p]),
    "tetris_verify_greedy_compact_f32": (
        C.c_int, [_p, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_sample_rows_f64": (C.c_int, [_p, _p, _p, _p, _p, _i32, _i32, _p, _p, _p, _p, _sz, _p]),
    "tetris_sample_rows_f32": (C.c_int, [_p, _p, _p, _p, _p, _i32, _i32, _p, _p, _p, _p, _sz, _p]),
    "tetris_residual_f64": (C.c_int, [_p, _p, _i32, _i32, _p, _p, _p, _p, _sz, _p]),
    "tetris_compact": (C.c_int, [_p, _p, _p, _p, _i32, _i32, _p, _p, _p]),
    "tetris_uniform_windows": (C.c_int, [_p, _i32, _i32, _i32, _p, _p, _p]),
    "tetris_sim_step": (
        C.c_int, [_p, _p, _i32, _i32, _i32, _i32, _i64, C.c_double, _p, _i64, _p, _i64, _p, _p, _p, _p, _p, _p, _p,
                  _p, _p, _p, _p, _p, _p, _p, _p]),
    "tetris_nccl_comm_info": (C.c_int, [_p, _p, _p]),
    "tetris_dist_gather_scores": (C.c_int, [_p, _p, _i32, _i32, _p, _p, _p, _p]),
    "tetris_dist_select_f64": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "tetris_dist_step_stochastic_f32": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _p, _p, _p, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                  _p, _p, _sz, _p]),
    "tetris_dist_step_stochastic_bf16": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                  _p, _p, _p, _p, _sz, _p]),
    "tetris_dist_step_greedy_f32": (
        C.c_int, [_p, _p, _i32, _i32, _i64, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _sz,
                  _p]),
}
EXPORTS = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = C.CDLL(str(LIB_PATH))
        except OSError as e:  # pragma: no cover - environment dependent
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def call(name: str, *args) -> None:
    """Invoke an ABI entry point; non-zero return codes raise (ValueError for argument errors)."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != OK:
        msg = lib.tetris_last_error().decode(errors="replace")
        if rc == INVALID_ARGUMENT:
            raise ValueError(msg)
        raise TetrisError(rc, msg)


def map_host(ptr: int, nbytes: int) -> int:
    """Device address of pinned (or newly registered) host memory, for zero-copy reads by the kernels."""
    out = C.c_void_p()
    call("tetris_map_host", ptr, nbytes, C.byref(out))
    return int(out.value)


def unmap_host(ptr: int) -> None:
    """Release a registration map_host made (no-op for caller-pinned memory)."""
    call("tetris_unmap_host", ptr)


def spec_max_requests() -> int:
    """Largest batch the speculative sampler takes on the current device (min(4096, 32 x SMs))."""
    return int(load().tetris_spec_max_requests())


def workspace_bytes(op: int, B: int, k: int, V: int) -> int:
    return int(load().tetris_workspace_bytes(op, B, k, V))
