"""Per-phase clock64() stamps of the selector's CTA 0 (select1_kernel layout: d0 start, d1 keys built, d2 radix done,
d3 windows, d4 epilogue; d9 = radix passes) for the cfg3 step, plus select-only timings."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2502_15197_b200 import _native as N  # noqa: E402
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

B, k, V, C = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (1024, 16, 128256, 8192)
bt = make_batch(B, k, V, seed=0)
step = ops.TetrisStep(B, k, V, C)
dbg = torch.zeros(64 + 32 * torch.cuda.get_device_properties(0).multi_processor_count, dtype=torch.int64, device='cuda')
N.load().tetris_debug_timestamps(dbg.data_ptr())
for it in range(5):
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    d = dbg.cpu().tolist()
    print('cycles: keys %d (staging %d) radix %d (passes %d) windows %d epilogue %d (accept wait %d) total %d' % (
        d[1] - d[0], d[5] - d[0], d[2] - d[1], d[9], d[3] - d[2], d[4] - d[3], d[6] - d[3], d[4] - d[0]))
    prev = d[1]
    parts = []
    for p in range(d[9]):
        h, pk, up = d[10 + 3 * p], d[11 + 3 * p], d[12 + 3 * p]
        parts.append('pass%d hist %d pick %d update %d' % (p, h - prev, pk - h, up - pk))
        prev = up
    print('   ', '; '.join(parts))
res = ops.select(bt.conf, C, bt.lengths)
for it in range(3):
    ops.select(bt.conf, C, bt.lengths, out=res)
    torch.cuda.synchronize()
    d = dbg.cpu().tolist()
    print('select-only cycles: keys %d (staging %d) radix %d (passes %d) windows %d total %d' % (
        d[1] - d[0], d[5] - d[0], d[2] - d[1], d[9], d[3] - d[2], d[3] - d[0]))
N.load().tetris_debug_timestamps(None)
torch.cuda.synchronize()
st = torch.cuda.Event(enable_timing=True)
en = torch.cuda.Event(enable_timing=True)
st.record()
for i in range(20):
    ops.select(bt.conf, C, bt.lengths, out=res)
en.record()
torch.cuda.synchronize()
print('select-only us (host-bound launches)', st.elapsed_time(en) / 20 * 1000)
