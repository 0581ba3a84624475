"""Timeline of one greedy step under graph replay: selector CTA 0 start/end (dbg[48..49]) and per-CTA stamps of
persist_greedy_kernel (0 entry, 1 first copy, 2 after griddepcontrol.wait, 3 last copy, 4 tail done).
usage: python tools/dbg_greedy.py [B k V C]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import _native as N  # noqa: E402
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

B, k, V, C = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (1024, 16, 128256, 8192)
bt = make_batch(B, k, V, seed=0, mode="greedy")
step = ops.TetrisStep(B, k, V, C, mode="greedy")
nsm = torch.cuda.get_device_properties(0).multi_processor_count
lib = N.load()
dbg = torch.zeros(64 + 32 * nsm, dtype=torch.int64, device="cuda")
run = lambda: step.run(bt.conf, bt.lengths, bt.p, None, bt.d)  # noqa: E731
run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        lib.tetris_debug_timestamps(dbg.data_ptr())
        run()
lib.tetris_debug_timestamps(None)
torch.cuda.current_stream().wait_stream(s)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
d = dbg.cpu()
st = d[64:64 + 8 * nsm].view(nsm, 8)
if int(d[48]):  # a separate selector launch stamped its CTA 0
    t0 = int(d[48])
    print("select %.2f -> %.2f us" % (0.0, (int(d[49]) - t0) / 1e3))
else:  # the one-launch step: the selection is the stream kernel's prologue
    t0 = int(st[:, 0][st[:, 0] > 0].min())
for j, name in enumerate(["entry", "first copy", "after wait", "last copy", "tail done"]):
    col = st[:, j][st[:, j] > 0]
    if len(col):
        rel = (col - t0).double() / 1e3
        print("%-11s min %8.2f median %8.2f max %8.2f us" % (name, rel.min(), rel.median(), rel.max()))
