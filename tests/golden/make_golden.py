"""Generate the golden vectors in tests/golden/ by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py
The reference package (tetris_sched 0.1.0, /root/reference/pkg/src) is imported read-only; nothing of it is copied.
Floats are stored as float.hex() strings so the fixtures are bit-exact.  The GPU box never runs this script; the
committed JSON files travel instead.
"""
from __future__ import annotations

import copy
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def H(x: float) -> str:
    return float(x).hex()


def main():
    sys.path.insert(0, str(REF))
    from tetris_sched.accept_model import (AcceptanceMatrix, DegenerateResidualError, TokenDistribution,
                                           emitted_law, residual_distribution, sample_emitted_token, verify_token)
    from tetris_sched.selector import Candidate, cumulative_products, expected_accepted, select_tetris
    from tetris_sched.sim_engine import apply_verification

    rng = np.random.default_rng(20260217)

    # ---- selection: cumulative_products + select_tetris (selector.py:95-176) --------------------------------------
    sel = []

    def add_sel(rows, capacity, tag):
        m = AcceptanceMatrix.from_rows(rows)
        cands = cumulative_products(m)
        s, st = select_tetris(cands, capacity)
        sel.append({"tag": tag, "rows": [[H(a) for a in r] for r in m.rows], "capacity": capacity,
                    "windows": list(s.windows), "stats": [st.extracts, st.inserts, st.peak_queue, st.comparisons],
                    "cum": [[H(c.cum) for c in r] for r in cands],
                    "expected_accepted": H(expected_accepted(s, m))})

    # the reference tests' KATs (test_selector.py:51-85)
    add_sel([[0.9, 0.9, 0.9], [0.5, 0.5]], 3, "kat_starve")
    add_sel([[0.9, 0.9, 0.9], [0.5, 0.5]], 4, "kat_fourth")
    add_sel([[0.7] * 3, [0.7] * 3], 4, "kat_equal")
    add_sel([[0.9], [0.5]], 0, "kat_c0")
    add_sel([[0.9], [0.5]], 10, "kat_exhaust")
    add_sel([[0.0, 0.0], [0.5]], 3, "kat_zero_fill")
    add_sel([[0.6] * 2] * 3, 1, "kat_row_tie")
    add_sel([[0.5, 0.0, 0.8]], 3, "kat_zero_tail")
    for i in range(300):  # test_selector.py:21-25 instance law
        n = int(rng.integers(1, 5))
        rows = [rng.random(int(rng.integers(1, 6))).tolist() for _ in range(n)]
        add_sel(rows, int(rng.integers(0, 9)), "random_small")
    for i in range(60):  # tie-heavy: quantised rates, exact 0/1, -0.0
        n = int(rng.integers(1, 24))
        k = int(rng.integers(1, 9))
        rows = []
        for _ in range(n):
            L = int(rng.integers(1, k + 1))
            r = (rng.integers(0, 9, L) / 8.0).tolist()
            r = [(-0.0 if (a == 0.0 and rng.random() < 0.5) else a) for a in r]
            rows.append(r)
        add_sel(rows, int(rng.integers(0, n * k + 2)), "ties")
    for (B, k) in [(64, 8), (200, 16)]:
        for C in (1, B, B * k // 3, B * k - 1):
            add_sel(rng.random((B, k)).tolist(), C, f"medium_{B}x{k}")
    # arbitrary (non-monotone) Candidate lists straight into select_tetris
    nonmono = []
    for i in range(80):
        n = int(rng.integers(1, 12))
        lists = []
        for r in range(n):
            L = int(rng.integers(0, 6))
            lists.append([Candidate(r, j + 1, float(rng.integers(0, 6) / 5.0)) for j in range(L)])
        C = int(rng.integers(0, 20))
        s, st = select_tetris(lists, C)
        nonmono.append({"cum": [[H(c.cum) for c in r] for r in lists], "capacity": C, "windows": list(s.windows),
                        "stats": [st.extracts, st.inserts, st.peak_queue, st.comparisons]})
    (OUT / "select.json").write_text(json.dumps({"monotone": sel, "candidates": nonmono}))

    # ---- verify_token (accept_model.py:291-313) -------------------------------------------------------------------
    vt = [{"ps": [H(0.2), H(0.8)], "pm": [H(0.5), H(0.5)], "token": 0, "u": H(0.999)},
          {"ps": [H(0.5), H(0.5)], "pm": [H(0.2), H(0.8)], "token": 0, "u": H(0.39)},
          {"ps": [H(0.5), H(0.5)], "pm": [H(0.2), H(0.8)], "token": 0, "u": H(0.41)}]
    for i in range(300):
        V = int(rng.integers(2, 40))
        ps = rng.dirichlet(np.ones(V))
        pm = rng.dirichlet(np.ones(V))
        t = int(rng.integers(0, V))
        u = float(rng.random())
        vt.append({"ps": [H(x) for x in ps], "pm": [H(x) for x in pm], "token": t, "u": H(u)})
    for c in vt:
        ps = TokenDistribution([float.fromhex(x) for x in c["ps"]])
        pm = TokenDistribution([float.fromhex(x) for x in c["pm"]])
        c["accepted"] = bool(verify_token(ps, pm, c["token"], float.fromhex(c["u"])))

    # ---- residual_distribution (accept_model.py:316-327) + emitted_law ---------------------------------------------
    res = []
    for (ps, pm) in [([0.5, 0.5], [0.2, 0.8]), ([0.25, 0.25, 0.5], [0.5, 0.25, 0.25]), ([0.3, 0.7], [0.3, 0.7])]:
        res.append((np.array(ps), np.array(pm)))
    for i in range(60):
        V = int([2, 3, 8, 64, 257, 512][i % 6])
        res.append((rng.dirichlet(np.ones(V)), rng.dirichlet(np.ones(V))))
    resid = []
    for ps, pm in res:
        a, b = TokenDistribution(ps), TokenDistribution(pm)
        entry = {"ps": [H(x) for x in a.probs], "pm": [H(x) for x in b.probs]}
        try:
            entry["residual"] = [H(x) for x in residual_distribution(a, b).probs]
        except DegenerateResidualError:
            entry["residual"] = None
        if a.vocab_size <= 64:
            entry["emitted_law"] = [H(x) for x in emitted_law(a, b).probs]
        resid.append(entry)

    # ---- Generator.choice == searchsorted(cumsum(p)/cumsum[-1], u, 'right'); sample_emitted_token --------------
    choice = []
    for i in range(200):
        V = int(rng.integers(2, 600))
        p = rng.dirichlet(np.ones(V) * float(rng.choice([0.05, 1.0])))
        g = np.random.default_rng(i)
        u = copy.deepcopy(g).random()
        choice.append({"p": [H(x) for x in p], "u": H(u), "index": int(g.choice(V, p=p))})
    chain = []
    for i in range(200):
        V = int(rng.integers(2, 9))
        ps = TokenDistribution(rng.dirichlet(np.ones(V)))
        pm = TokenDistribution(rng.dirichlet(np.ones(V)))
        g = np.random.default_rng(1000 + i)
        us = copy.deepcopy(g).random(3)
        tok, acc = sample_emitted_token(ps, pm, g)
        chain.append({"ps": [H(x) for x in ps.probs], "pm": [H(x) for x in pm.probs], "seed": 1000 + i,
                      "u": [H(x) for x in us], "token": tok, "accepted": bool(acc)})
    (OUT / "token.json").write_text(json.dumps({"verify_token": vt, "residual": resid, "choice": choice,
                                                "chain": chain}))

    # ---- apply_verification (sim_engine.py:374-404) ---------------------------------------------------------------
    from tetris_sched.selector import Selection

    av = []
    for i in range(200):
        n = int(rng.integers(1, 20))
        rows = [rng.random(int(rng.integers(1, 8))).tolist() for _ in range(n)]
        truth = AcceptanceMatrix.from_rows(rows)
        w = [int(rng.integers(0, len(r) + 1)) for r in rows]
        seed = 5000 + i
        draws = copy.deepcopy(np.random.default_rng(seed)).random(sum(w))
        acc = apply_verification(Selection(tuple(w)), truth, np.random.default_rng(seed))
        av.append({"rows": [[H(a) for a in r] for r in rows], "windows": w, "seed": seed,
                   "draws": [H(x) for x in draws], "accepted": list(acc)})
    (OUT / "verify_matrix.json").write_text(json.dumps(av))
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
