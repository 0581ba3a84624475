"""Launch-mode experiment: the same step eager, as one CUDA graph per step, and as one graph of 8 steps.
usage: python tools/exp_launch.py [B k V C mode]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

a = sys.argv[1:]
B, k, V, C = (int(x) for x in a[:4]) if len(a) >= 4 else (1024, 16, 128256, 8192)
mode = a[4] if len(a) >= 5 else "stochastic"
sets = [make_batch(B, k, V, seed=s, mode=mode) for s in range(2)]
step = ops.TetrisStep(B, k, V, C, mode=mode)
run = lambda s: step.run(s.conf, s.lengths, s.p, s.q, s.d, s.u_acc, s.u_res)  # noqa: E731


def timed(fn, n):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


def capture(nsteps, first):
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        for j in range(nsteps):
            run(sets[(first + j) % 2])
    torch.cuda.current_stream().wait_stream(cs)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for j in range(nsteps):
            run(sets[(first + j) % 2])
    return g


g1 = [capture(1, s) for s in range(2)]
g8 = capture(8, 0)
n = 400
print("eager          %.2f us/step" % timed(lambda i: run(sets[i % 2]), n))
print("graph x1       %.2f us/step" % timed(lambda i: g1[i % 2].replay(), n))
print("graph x8       %.2f us/step" % (timed(lambda i: g8.replay(), n // 8) / 8))
