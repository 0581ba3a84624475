"""Debug: one-launch (fused) vs two-launch step on one batch; prints the rows whose windows / accepted lengths differ.
usage: python tools/dbg_fused.py [B k V C]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from test_fused_step import _run  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

B, k, V, C = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (256, 8, 32000, 1024)
bt = make_batch(B, k, V, seed=B * 31 + k)
args = (bt.conf, bt.lengths, B, k, C, 0, B, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res, V, None)
one = _run(*args, fused=True).results()
two = _run(*args, fused=False).results()
for name in one:
    if not np.array_equal(one[name], two[name]):
        idx = np.nonzero(one[name] != two[name])[0] if one[name].shape == two[name].shape else []
        print(name, "differs at", idx[:20], "fused", one[name][idx[:20]], "two", two[name][idx[:20]])
w1, w2 = one["windows"], two["windows"]
print("sum windows fused %d two %d (C=%d)" % (w1.sum(), w2.sum(), C))
