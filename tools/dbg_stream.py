"""Per-CTA %globaltimer stamps of persist_stream_kernel (slots: 0 entry, 1 after griddepcontrol.wait, 2 first copy
issued, 3 last copy issued, 4 first stage consumed, 5 publisher done, 6 descents done, 7..12 the speculative / fused
prologue) for one step of a config.
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
dbg = torch.zeros(64 + 32 * nsm, dtype=torch.int64, device="cuda")
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
d = dbg[64:64 + 16 * nsm].view(nsm, 16).cpu()
cyc = dbg[64 + 16 * nsm:].view(nsm, 16).cpu()
t0 = int(d[:, 0][d[:, 0] > 0].min())
names = ["entry", "after wait", "first copy", "last copy", "first consumed", "publisher done", "descents done",
         "spec prologue / fused: first item ready (producer)", "fused: scores loaded", "fused: keys built",
         "fused: ranks done", "fused: last CTA publishes", "fused: scans released",
         "descent (warp 0): request's chunks counted", "descent (warp 0): done", "descent (warp 0): sums in"]
for s, nme in enumerate(names):
    col = d[:, s]
    col = col[col > 0]
    if len(col) == 0:
        continue
    rel = (col - t0).double() / 1e3
    print("%-52s min %7.2f  median %7.2f  max %7.2f us (CTAs %d)" % (nme, rel.min(), rel.median(), rel.max(), len(col)))

# in-CTA phase lengths in SM cycles (clock64 beside each stamp): consecutive slots of the fused prologue
for a_, b_, nme in ((1, 8, "wait -> scores loaded"), (8, 9, "scores -> keys"), (9, 10, "keys -> ranks+verdicts"),
                    (10, 11, "ranks -> published (last CTA)"), (11, 12, "published -> scans released (last CTA)"),
                    (1, 7, "wait -> first item ready"), (7, 2, "ready -> first copy"),
                    (2, 3, "first -> last copy"), (3, 5, "last copy -> publisher done"),
                    (5, 6, "publisher done -> descents done"), (5, 13, "publisher done -> warp 0 request counted"),
                    (13, 15, "counted -> descent sums in"), (15, 14, "sums in -> descent done")):
    m = (cyc[:, a_] > 0) & (cyc[:, b_] > 0)
    if m.sum() == 0:
        continue
    dc = (cyc[m, b_] - cyc[m, a_]).double()
    print("cycles %-40s min %8.0f  median %8.0f  max %8.0f (CTAs %d)" % (nme, dc.min(), dc.median(), dc.max(), int(m.sum())))

# the latest CTAs (their descents end the step): every stamp, us from the first entry
late = torch.argsort(d[:, 6], descending=True)[:6]
print("latest CTAs (cta: entry, after wait, first copy, last copy, first consumed, publisher done, descents done, "
      "warp-0 request counted / sums in / done):")
for c in late.tolist():
    row = d[c]
    f = lambda s: "%.2f" % ((int(row[s]) - t0) / 1e3) if int(row[s]) > 0 else "-"  # noqa: E731
    print("  %3d: %s" % (c, " ".join(f(s) for s in (0, 1, 2, 3, 4, 5, 6, 13, 15, 14))))
