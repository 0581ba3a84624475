import sys, torch
sys.path.insert(0, '.')
from paper_2502_15197_b200 import ops, _native as N
from paper_2502_15197_b200.synthetic import make_batch
B,k,V,C = 1024,16,128256,8192
bt = make_batch(B,k,V,seed=0)
step = ops.TetrisStep(B,k,V,C)
dbg = torch.zeros(32, dtype=torch.int64, device='cuda')
N.load().tetris_debug_timestamps(dbg.data_ptr())
for it in range(5):
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    d = dbg.cpu().tolist()
    print('phase cycles: p0 %d scan %d radix %d (passes %d) windows %d accept %d compact %d' % (d[1]-d[0], d[2]-d[1], d[3]-d[2], d[9], d[4]-d[3], d[5]-d[4], d[6]-d[5]))
# select only (no epilogue)
res = ops.select(bt.conf, C, bt.lengths); torch.cuda.synchronize()
for it in range(3):
    res = ops.select(bt.conf, C, bt.lengths); torch.cuda.synchronize()
    d = dbg.cpu().tolist()
    print('select-only: p0 %d [stage %d sync %d rows %d] scan %d radix %d (passes %d) windows %d' % (d[1]-d[0], d[10]-d[0], d[11]-d[10], d[12]-d[11], d[2]-d[1], d[3]-d[2], d[9], d[4]-d[3]))
st=torch.cuda.Event(enable_timing=True); en=torch.cuda.Event(enable_timing=True)
st.record()
for i in range(20): ops.select(bt.conf, C, bt.lengths)
en.record(); torch.cuda.synchronize(); print('select-only us', st.elapsed_time(en)/20*1000)
