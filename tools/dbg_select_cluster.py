"""Per-phase clock64() stamps of the large-batch selector (B*k > 16384) for a select-only call."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2502_15197_b200 import _native as N  # noqa: E402
from paper_2502_15197_b200 import ops  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
k, C = 16, int(sys.argv[2]) if len(sys.argv) > 2 else 131072
g = torch.Generator(device="cuda").manual_seed(0)
conf = (torch.rand(B, k, dtype=torch.float64, device="cuda", generator=g) ** 0.3).contiguous()
dbg = torch.zeros(64 + 32 * torch.cuda.get_device_properties(0).multi_processor_count, dtype=torch.int64, device="cuda")
N.load().tetris_debug_timestamps(dbg.data_ptr())
res = ops.select(conf, C)
for it in range(4):
    ops.select(conf, C, out=res)
    torch.cuda.synchronize()
    d = dbg.cpu().tolist()
    print('cycles: p0 %d scan %d radix %d (passes %d) windows %d total %d' % (
        d[1] - d[0], d[2] - d[1], d[3] - d[2], d[9], d[4] - d[3], d[4] - d[0]))
    prev = d[2]
    parts = []
    for p in range(min(d[9], 3)):
        s = d[10 + 5 * p: 15 + 5 * p]
        parts.append('p%d copy %d pick %d update %d count %d barrier %d' % (p, s[0] - prev, s[1] - s[0], s[2] - s[1],
                                                                          s[3] - s[2], s[4] - s[3]))
        prev = s[4]
    print('   ', '; '.join(parts))
N.load().tetris_debug_timestamps(None)
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ops.select(conf, C, out=res)
torch.cuda.synchronize()
st.record()
for i in range(50):
    ops.select(conf, C, out=res)
en.record()
torch.cuda.synchronize()
print('select us (host-bound launches)', st.elapsed_time(en) / 50 * 1000)
