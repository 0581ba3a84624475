"""Seeded, numpy-only input recipes for the configuration-scale selection goldens (test infrastructure).

Shared by make_golden_scale.py (which runs the REFERENCE on them in the build container) and the GPU tests (which
regenerate the same matrices on the box and check their sha256 before comparing)."""
from __future__ import annotations

import hashlib

import numpy as np

# (tag, B, k, capacities, recipe, seed) -- BASELINE.json configs[0..4] shapes (SURVEY.md §8 cfg table)
CASES = [
    ("cfg1", 16, 5, [48], "beta", 11),
    ("cfg1_ragged", 16, 5, [48, 30], "beta_ragged", 12),
    ("cfg2", 256, 8, [1024], "beta", 21),
    ("cfg2_ties", 256, 8, [1024, 777], "ties", 22),
    ("cfg3", 1024, 16, [8192], "beta", 31),
    ("cfg3_ties", 1024, 16, [8192, 5000], "ties", 32),
    ("cfg3_ragged", 1024, 16, [8192], "beta_ragged", 33),
    ("cfg4", 4096, 16, [4096, 8192, 16384, 32768, 65536], "beta", 41),
    ("cfg4_ties", 4096, 16, [4096, 65536], "ties", 42),
    ("cfg5", 16384, 16, [131072], "beta", 51),
]


def conf_matrix(B: int, k: int, recipe: str, seed: int):
    """Acceptance-rate matrix [B, k] f64 and row lengths [B] (ragged rows: entries past the length are 0)."""
    rng = np.random.default_rng(seed)
    if recipe in ("beta", "beta_ragged"):
        # two-population mix like MixSource (accept_model.py:134-158): easy rows near 1, hard rows spread out
        easy = rng.random(B) < 0.5
        a = np.where(easy[:, None], rng.beta(8.0, 1.0, (B, k)), rng.beta(1.5, 1.5, (B, k)))
    elif recipe == "ties":
        # quantised rates (multiples of 1/16 incl. exact 0 and 1) and -0.0: heavy cum / row / depth ties
        a = rng.integers(0, 17, (B, k)) / 16.0
        neg = (a == 0.0) & (rng.random((B, k)) < 0.5)
        a[neg] = -0.0
    else:
        raise ValueError(recipe)
    lengths = np.full(B, k, np.int32)
    if recipe.endswith("ragged"):
        lengths = rng.integers(1, k + 1, B).astype(np.int32)
        a[np.arange(k)[None, :] >= lengths[:, None]] = 0.0
    return np.ascontiguousarray(a, np.float64), lengths


def rows_of(a, lengths):
    return [a[i, : lengths[i]].tolist() for i in range(a.shape[0])]


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def enc_windows(w) -> str:
    return "".join(np.base_repr(int(x), 36) for x in w)


def dec_windows(s: str):
    return np.array([int(c, 36) for c in s], np.int32)
