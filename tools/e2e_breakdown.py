"""Where the host-buffer (e2e) step's time goes: cfg3 through ops.HostTetrisStep, events around each whole step, plus
(under `ncu --metrics gpu__time_duration.sum`) the per-kernel durations of the same calls.
usage: python tools/e2e_breakdown.py [steps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
B, k, V, C = 1024, 16, 128256, 8192
bt = make_batch(B, k, V, seed=0)
p_h = torch.empty(bt.p.shape, dtype=bt.p.dtype, pin_memory=True)
p_h.copy_(bt.p)
q_h = torch.empty(bt.q.shape, dtype=bt.q.dtype, pin_memory=True)
q_h.copy_(bt.q)
small = [t.cpu().pin_memory() for t in (bt.conf, bt.lengths, bt.d, bt.u_acc, bt.u_res)]
del bt
hs = ops.HostTetrisStep(B, k, V, C, p_h, q_h)
for _ in range(2):
    hs.run(*small)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for a, b in ev:
    a.record()
    hs.run(*small)
    b.record()
torch.cuda.synchronize()
print("e2e step ms:", ["%.3f" % a.elapsed_time(b) for a, b in ev], "tokens", int(hs.offsets_host[-1]))
