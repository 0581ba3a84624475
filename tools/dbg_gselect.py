"""Per-phase clock64() stamps of gselect_kernel's CTA 0 (d0 start, d1 keys + pass-0 histogram published, d2 after the
first grid barrier, per pass p: d[10+5p] histogram copied, d[11+5p] digit picked, d[12+5p] ranges updated, d[13+5p]
next histogram built, d[14+5p] after the pass's grid barrier; d3 radix done, d9 passes) for a selection-only call.
usage: python tools/dbg_gselect.py [B k C]"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2502_15197_b200 import _native as N  # noqa: E402
from paper_2502_15197_b200 import ops  # noqa: E402

B, k, C = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (4096, 16, 8192)
g = torch.Generator(device="cpu").manual_seed(1)
conf = (torch.rand(B, k, dtype=torch.float64, generator=g) ** 0.25).cuda()
dbg = torch.zeros(64 + 32 * torch.cuda.get_device_properties(0).multi_processor_count, dtype=torch.int64, device='cuda')
res = ops.select(conf, C)
lib = N.load()
for it in range(4):
    lib.tetris_debug_timestamps(dbg.data_ptr() if it == 3 else None)
    ops.select(conf, C, out=res)
    torch.cuda.synchronize()
lib.tetris_debug_timestamps(None)
d = dbg.cpu().tolist()
print("cycles: keys+hist0 %d, barrier0 %d, radix %d (passes %d), after radix -> end n/a" % (
    d[1] - d[0], d[2] - d[1], d[3] - d[2], d[9]))
prev = d[2]
for p in range(d[9]):
    s = [d[10 + 5 * p + i] for i in range(5)]
    parts = ["copy %d" % (s[0] - prev), "pick %d" % (s[1] - s[0])]
    if s[2]:
        parts += ["update %d" % (s[2] - s[1])]
    if s[3]:
        parts += ["hist %d" % (s[3] - s[2]), "publish+barrier %d" % (s[4] - s[3])]
    print("  pass %d: %s" % (p, ", ".join(parts)))
    prev = s[4] if s[4] else s[1]
# graph-replayed select-only time
gr = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    ops.select(conf, C, out=res, stream=s)
    with torch.cuda.graph(gr, stream=s):
        for _ in range(20):
            ops.select(conf, C, out=res, stream=s)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    gr.replay()
e1.record()
torch.cuda.synchronize()
print("select-only us (graph, same input, L2-warm): %.2f" % (e0.elapsed_time(e1) / 200 * 1000))
