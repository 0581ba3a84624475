"""Greedy step timeline under CUDA-graph replay: per-CTA %globaltimer stamps of persist_greedy_kernel (slots: 0 entry,
1 first copy, 2 after griddepcontrol.wait, 3 last copy, 4 tail done, 6 last CTA elected, 7 its compaction done) for one replay of a 2-step graph, so the gap
between consecutive steps shows.  usage: python tools/dbg_graph_greedy.py [B k V C]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import _native as N  # noqa: E402
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

B, k, V, C = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (16, 5, 32000, 48)
bt = make_batch(B, k, V, seed=0, mode="greedy")
step = ops.TetrisStep(B, k, V, C, mode="greedy")
nsm = torch.cuda.get_device_properties(0).multi_processor_count
lib = N.load()
dbgs = [torch.zeros(64 + 32 * nsm, dtype=torch.int64, device="cuda") for _ in range(2)]
run = lambda: step.run(bt.conf, bt.lengths, bt.p, None, bt.d)  # noqa: E731
run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for i in range(2):
            lib.tetris_debug_timestamps(dbgs[i].data_ptr())
            run()
lib.tetris_debug_timestamps(None)
torch.cuda.current_stream().wait_stream(s)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(50):
    g.replay()
ev[1].record()
torch.cuda.synchronize()
print("graph of 2 steps: %.2f us per step" % (ev[0].elapsed_time(ev[1]) * 1e3 / 100))
t0 = None
for i, d in enumerate(dbgs):
    st = d.cpu()[64:64 + 8 * nsm].view(nsm, 8)
    col = lambda j: st[:, j][st[:, j] > 0].double()  # noqa: E731
    if t0 is None:
        t0 = float(col(0).min())
    rel = lambda x: (x - t0) / 1e3  # noqa: E731
    print("step %d: entry %.2f (median %.2f, max %.2f) | after wait median %.2f | first copy median %.2f | last copy "
          "max %.2f | tail done median %.2f max %.2f" % (
              i, rel(col(0).min()), rel(col(0).median()), rel(col(0).max()), rel(col(2).median()),
              rel(col(1).median()), rel(col(3).max()), rel(col(4).median()), rel(col(4).max())))
    if len(col(6)):
        print("        last CTA elected %.2f, its scans + compaction done %.2f" % (rel(col(6).max()), rel(col(7).max())))
    print("        per slot (min / median / max over CTAs):",
          " ".join("s%d %.2f/%.2f/%.2f" % (j, rel(col(j).min()), rel(col(j).median()), rel(col(j).max()))
                   for j in range(8) if len(col(j))))
    print("        CTA 0:", " ".join("s%d %.2f" % (j, rel(float(st[0, j]))) for j in range(8) if int(st[0, j]) > 0))
