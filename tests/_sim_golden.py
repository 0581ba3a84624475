"""Loader of tests/golden/sim.json (reference simulator traces, tests/golden/make_golden_sim.py)."""
import base64
import json
from pathlib import Path

import numpy as np

PATH = Path(__file__).resolve().parent / "golden" / "sim.json"


def dec(s, dtype):
    return np.frombuffer(base64.b64decode(s), dtype=dtype)


def runs():
    out = []
    for r in json.loads(PATH.read_text())["runs"]:
        K = r["k"] + r["extra"]
        B = r["batch_size"]
        steps = []
        for s in r["steps"]:
            tm = dec(s["truth"], "<f8").reshape(B, K)
            sm = dec(s["surrogate"], "<f8").reshape(B, K)
            d = s["depths"]
            steps.append(dict(s, truth_rows=[list(tm[i, :d[i]]) for i in range(B)],
                              surrogate_rows=[list(sm[i, :d[i]]) for i in range(B)],
                              expected=float.fromhex(s["expected_accepted"]), alpha=float.fromhex(s["alpha_hat"])))
        out.append(dict(r, lengths=dec(r["lengths"], "<i4"), uniforms=dec(r["uniforms"], "<f8"), steps=steps))
    return out
