"""Configuration-scale selection goldens produced by running the REFERENCE itself (tetris_sched 0.1.0).

    python tests/golden/make_golden_scale.py        # build container only (needs /root/reference)

For each case of scale_inputs.CASES (cfg1..cfg5 shapes, incl. quantised-tie and ragged variants and the cfg4
capacity sweep) this records what the reference's own functions return on the seeded matrix:
`cumulative_products` (selector.py:95-110; sha256 of every cum bit), `select_tetris` (selector.py:133-176; the
windows and the full PolicyStats incl. heapq `comparisons`) and `expected_accepted` (selector.py:286-306, float.hex).
tests/test_golden_scale.py checks the GPU selection against these, bit for bit.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from scale_inputs import CASES, conf_matrix, enc_windows, rows_of, sha  # noqa: E402


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from tetris_sched.accept_model import AcceptanceMatrix
    from tetris_sched.selector import cumulative_products, expected_accepted, select_tetris

    out = []
    for tag, B, k, caps, recipe, seed in CASES:
        a, lengths = conf_matrix(B, k, recipe, seed)
        m = AcceptanceMatrix.from_rows(rows_of(a, lengths))
        t0 = time.perf_counter()
        cands = cumulative_products(m)
        cum = np.zeros((B, k), np.float64)
        for i, r in enumerate(cands):
            cum[i, : len(r)] = [c.cum for c in r]
        t_cum = time.perf_counter() - t0
        for C in caps:
            t0 = time.perf_counter()
            s, st = select_tetris(cands, C)
            t_sel = time.perf_counter() - t0
            out.append({"tag": tag, "B": B, "k": k, "C": C, "recipe": recipe, "seed": seed,
                        "conf_sha256": sha(a), "lengths_sha256": sha(lengths), "cum_sha256": sha(cum),
                        "windows": enc_windows(s.windows),
                        "stats": [st.extracts, st.inserts, st.peak_queue, st.comparisons],
                        "expected_accepted": float(expected_accepted(s, m)).hex(),
                        "ref_seconds": {"cumulative_products": round(t_cum, 4), "select_tetris": round(t_sel, 4)}})
            print(tag, B, k, C, st, f"{t_cum:.3f}s {t_sel:.3f}s")
    (HERE / "select_scale.json").write_text(json.dumps({"generator": "tetris_sched 0.1.0 (/root/reference/pkg)",
                                                        "numpy": np.__version__, "cases": out}, indent=0))


if __name__ == "__main__":
    main()
