"""B200-native TETRIS batch speculative-decoding hot path (arXiv 2502.15197).

Layers: csrc/ (sm_100a kernels + C ABI, include/tetris_b200.h) -> _native (ctypes) -> ops (batched tensor API)
-> selector / accept_model / sim_engine (drop-in adapters with the reference package's names and semantics)
-> dist (request-sharded multi-GPU selection).
"""
__version__ = "0.1.0"

from . import errors  # noqa: F401
