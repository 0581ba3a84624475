"""Small runs of every product kernel for compute-sanitizer (memcheck / racecheck / synccheck):
python tools/sanitize.py  — exercises the speculative and plain samplers, the greedy stream, both selectors."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import ops  # noqa: E402
from paper_2502_15197_b200.synthetic import make_batch  # noqa: E402

for (B, k, V, C, mode) in [(300, 6, 16384, 900, "stochastic"), (64, 4, 8200, 10, "stochastic"),
                           (200, 8, 8200, 700, "greedy"), (2048, 9, 1024, 9000, "greedy"),
                           (37, 0, 8192, 5, "stochastic"), (37, 0, 8192, 5, "greedy"),  # nothing drafted
                           (90, 5, 1003, 200, "stochastic"), (90, 5, 1003, 200, "greedy"),  # V % 8 != 0
                           (16, 5, 32000, 48, "greedy"),  # cfg1: one launch, CTA 0 finishes <= 36 requests alone
                           (256, 8, 32000, 1200, "stochastic")]:  # cfg2 shape: the one-launch step at 2048 cells
    bt = make_batch(B, k, V, seed=1, mode=mode, ragged=True)
    step = ops.TetrisStep(B, k, V, C, mode=mode)
    for _ in range(2):
        step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
# the speculative sampler explicitly (the step only picks it for >= 4096 streamed chunks)
from paper_2502_15197_b200 import _native as N  # noqa: E402
B, k, V, C = 300, 6, 16384, 900
bt = make_batch(B, k, V, seed=2, ragged=True)
step = ops.TetrisStep(B, k, V, C)
lib = N.load()
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    assert lib.tetris_select_accept_f32(bt.conf.data_ptr(), bt.lengths.data_ptr(), B, k, C, 0, B, bt.p.data_ptr(),
                                        bt.q.data_ptr(), bt.d.data_ptr(), bt.u_acc.data_ptr(), 0, None, V,
                                        step.windows_all.data_ptr(), step.win_offsets.data_ptr(),
                                        step.accepted.data_ptr(), step.offsets.data_ptr(), step.tokens.data_ptr(),
                                        step.stats.data_ptr(), step.status.data_ptr(), step.ws.ptr, step.ws.nbytes,
                                        s) == 0
    assert lib.tetris_resample_spec_f32(bt.p.data_ptr(), bt.q.data_ptr(), bt.u_res.data_ptr(), bt.u_acc.data_ptr(),
                                        bt.lengths.data_ptr(), B, k, V, bt.d.data_ptr(), step.accepted.data_ptr(),
                                        step.offsets.data_ptr(), step.out_tok.data_ptr(), step.mass.data_ptr(),
                                        step.tokens.data_ptr(), step.status.data_ptr(), step.ws.ptr, step.ws.nbytes,
                                        s) == 0
torch.cuda.synchronize()
ops.raise_for_status(step.status)
print("ok")
# round 2: the logits form (fused one-launch and two-launch sizes), the host-buffer steps (row-gather kernels), the grid
# selector's clamped first pass on a stochastic step, the GPU simulator step
from paper_2502_15197_b200.synthetic import make_logit_batch  # noqa: E402

for (B, k, V, C) in [(200, 8, 8192, 700), (600, 8, 8192, 2000)]:
    lb = make_logit_batch(B, k, V, seed=3, ragged=True)
    step = ops.TetrisStep(B, k, V, C)
    for _ in range(2):
        step.run_logits(lb.conf, lb.lengths, lb.zp, lb.lse_p, lb.zq, lb.lse_q, lb.d, lb.u_acc, lb.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
for mode in ("stochastic", "greedy"):
    B, k, V, C = 96, 5, 8192, 300
    bt = make_batch(B, k, V, seed=4, mode=mode, ragged=True)
    hs = ops.HostTetrisStep(B, k, V, C, bt.p.cpu().pin_memory(),
                            bt.q.cpu().pin_memory() if mode == "stochastic" else None, mode=mode)
    small = [t.cpu().pin_memory() for t in (bt.conf, bt.lengths, bt.d, bt.u_acc, bt.u_res)]
    for _ in range(2):
        hs.run(*(small if mode == "stochastic" else small[:3]))
    torch.cuda.synchronize()
    ops.raise_for_status(hs.step.status)
B, k, V, C = 2048, 16, 2048, 12000  # 32768 cells: grid selector + speculative sampler
bt = make_batch(B, k, V, seed=5, ragged=True)
step = ops.TetrisStep(B, k, V, C)
for _ in range(2):
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
torch.cuda.synchronize()
ops.raise_for_status(step.status)
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from _sim_golden import runs  # noqa: E402
from paper_2502_15197_b200.sim_engine import GpuSimulator  # noqa: E402

run = runs()[0]
sim = GpuSimulator(run["batch_size"], run["k"], run["capacity"], extra=run["extra"], policy=run["policy"],
                   uniforms=run["uniforms"], lengths=run["lengths"], device="cuda")
for s_ in run["steps"][:3]:
    sim.step(s_["truth_rows"], s_["surrogate_rows"])
print("sanitize.py: all kernels ran")
