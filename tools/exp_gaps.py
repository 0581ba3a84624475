"""Experiment: where does the time between the step's kernels go?  Times (CUDA events, eager) N back-to-back
select_accept launches, N back-to-back resample launches, and N alternating pairs (the real step)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

# optional argv: B k V C (default cfg3)
B, k, V, C = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (1024, 16, 128256, 8192)
bt = make_batch(B, k, V, seed=0)
step = ops.TetrisStep(B, k, V, C)
lib, ws = step._lib, step.ws


def sel():
    s = torch.cuda.current_stream().cuda_stream
    lib.tetris_select_accept_f32(bt.conf.data_ptr(), bt.lengths.data_ptr(), B, k, C, 0, B, bt.p.data_ptr(),
                                 bt.q.data_ptr(), bt.d.data_ptr(), bt.u_acc.data_ptr(), 0, None, V,
                                 step.windows_all.data_ptr(), step.win_offsets.data_ptr(), step.accepted.data_ptr(),
                                 step.offsets.data_ptr(), step.tokens.data_ptr(), step.stats.data_ptr(),
                                 step.status.data_ptr(), ws.ptr, ws.nbytes, s)


def sel_only():
    s = torch.cuda.current_stream().cuda_stream
    lib.tetris_select_f64(bt.conf.data_ptr(), bt.lengths.data_ptr(), B, k, C, 0, step.windows_all.data_ptr(),
                          step.win_offsets.data_ptr(), None, step.stats.data_ptr(), step.status.data_ptr(), ws.ptr,
                          ws.nbytes, s)


def res():
    s = torch.cuda.current_stream().cuda_stream
    lib.tetris_resample_f32(bt.p.data_ptr(), bt.q.data_ptr(), bt.u_res.data_ptr(), B, k, V, bt.d.data_ptr(),
                            step.accepted.data_ptr(), step.offsets.data_ptr(), step.out_tok.data_ptr(),
                            step.mass.data_ptr(), step.tokens.data_ptr(), step.status.data_ptr(), ws.ptr, ws.nbytes, s)


def timeit(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


print("select_accept back-to-back  %.2f us" % timeit(sel))
print("resample back-to-back       %.2f us" % timeit(res))
print("select+resample (step)      %.2f us" % timeit(lambda: (sel(), res())))
gs = graph_of(sel)
gr = graph_of(res)
g2 = graph_of(lambda: (sel(), res()))
print("graph select                %.2f us" % timeit(gs.replay))
print("graph select only (no accept epilogue) %.2f us" % timeit(graph_of(sel_only).replay))
print("graph resample              %.2f us" % timeit(gr.replay))
print("graph step                  %.2f us" % timeit(g2.replay))
x = torch.empty(1 << 20, device="cuda")
print("tiny torch kernel           %.2f us" % timeit(lambda: x.add_(1.0)))
print("select + tiny               %.2f us" % timeit(lambda: (sel(), x.add_(1.0))))
print("resample + tiny             %.2f us" % timeit(lambda: (res(), x.add_(1.0))))


def seq(fns, n=20):
    """events between consecutive launches of the sequence; returns mean us per segment"""
    for _ in range(3):
        for f in fns:
            f()
    torch.cuda.synchronize()
    tot = [0.0] * len(fns)
    for _ in range(n):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(fns) + 1)]
        ev[0].record()
        for i, f in enumerate(fns):
            f()
            ev[i + 1].record()
        torch.cuda.synchronize()
        for i in range(len(fns)):
            tot[i] += ev[i].elapsed_time(ev[i + 1]) * 1e3 / n
    return " | ".join("%.1f" % t for t in tot)


tiny = lambda: x.add_(1.0)  # noqa: E731
print("seq res,tiny,sel,res,sel,sel,tiny,tiny:", seq([res, tiny, sel, res, sel, sel, tiny, tiny]))
torch.cuda.synchronize()
import time  # noqa: E402
t = time.perf_counter()
for _ in range(100):
    sel()
print("host us per sel() call %.1f" % ((time.perf_counter() - t) * 1e4))
t = time.perf_counter()
for _ in range(100):
    tiny()
print("host us per tiny call %.1f" % ((time.perf_counter() - t) * 1e4))
torch.cuda.synchronize()
