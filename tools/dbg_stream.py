"""Per-CTA %globaltimer stamps of persist_stream_kernel (slots: 0 entry, 1 after griddepcontrol.wait, 2 first copy
issued, 3 last copy issued, 4 first stage consumed, 5 publisher done, 6 descents done) for one step of a config.
usage: python tools/dbg_stream.py [B k V C]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import _native as N  # noqa: E402
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch, make_logit_batch  # noqa: E402

serial = "--serial" in sys.argv  # events between the launches: the sampler does not overlap the selector
logits = "--logits" in sys.argv  # the logits form (bf16 rows + lse)
argv = [x for x in sys.argv[1:] if not x.startswith("--")]
B, k, V, C = (int(x) for x in argv[:4]) if len(argv) >= 4 else (1024, 16, 128256, 8192)
bt = make_logit_batch(B, k, V, seed=0) if logits else make_batch(B, k, V, seed=0)
step = ops.TetrisStep(B, k, V, C)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
dbg = torch.zeros(64 + 8 * nsm, dtype=torch.int64, device="cuda")
lib = N.load()
for it in range(4):
    lib.tetris_debug_timestamps(dbg.data_ptr() if it == 3 else None)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if serial else None
    if logits:
        step.run_logits(bt.conf, bt.lengths, bt.zp, bt.lse_p, bt.zq, bt.lse_q, bt.d, bt.u_acc, bt.u_res, events=evs)
    else:
        step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res, events=evs)
    torch.cuda.synchronize()
lib.tetris_debug_timestamps(None)
d = dbg[64:].view(nsm, 8).cpu()
t0 = int(d[:, 0][d[:, 0] > 0].min())
names = ["entry", "after wait", "first copy", "last copy", "first consumed", "publisher done", "descents done",
         "spec prologue"]
for s, nme in enumerate(names):
    col = d[:, s]
    col = col[col > 0]
    if len(col) == 0:
        continue
    rel = (col - t0).double() / 1e3
    print("%-15s min %7.2f  median %7.2f  max %7.2f us (CTAs %d)" % (nme, rel.min(), rel.median(), rel.max(), len(col)))
