"""Step timeline under CUDA-graph replay (the bench's launch mode): %globaltimer stamps of the selector (CTA 0 start /
end, dbg[48..49]) and of the sampler's CTAs (dbg[64 + 16 cta + slot]) for one replay of a 2-step graph, so the gaps
between kernels and between steps show.  usage: python tools/dbg_graph.py [B k V C]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import _native as N  # noqa: E402
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

B, k, V, C = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (1024, 16, 128256, 8192)
bt = make_batch(B, k, V, seed=0)
step = ops.TetrisStep(B, k, V, C)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
lib = N.load()
dbgs = [torch.zeros(64 + 32 * nsm, dtype=torch.int64, device="cuda") for _ in range(2)]
run = lambda: step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)  # noqa: E731
run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for i in range(2):  # each step's kernels write their own debug buffer (captured launch parameters)
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
    d = d.cpu()
    sel0, sel1 = int(d[48]), int(d[49])
    st = d[64:64 + 16 * nsm].view(nsm, 16)
    if sel0 == 0:  # the one-launch step (the selection is the sampler's prologue): time from the first CTA entry
        sel0 = sel1 = int(st[:, 0][st[:, 0] > 0].min())
    t0 = sel0 if t0 is None else t0
    rel = lambda x: (x - t0) / 1e3  # noqa: E731
    col = lambda j: st[:, j][st[:, j] > 0]  # noqa: E731
    print("step %d: select %.2f -> %.2f us | sampler entry %.2f (median %.2f, max %.2f) | first copy %.2f | last "
          "descent %.2f (median CTA %.2f)"
          % (i, rel(sel0), rel(sel1), rel(int(col(0).min())), rel(float(col(0).double().median())),
             rel(int(col(0).max())), rel(float(col(2).double().median())), rel(int(col(6).max())),
             rel(float(col(6).double().median()))))
