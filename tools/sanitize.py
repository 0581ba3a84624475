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
                           (90, 5, 1003, 200, "stochastic"), (90, 5, 1003, 200, "greedy")]:  # V % 8 != 0
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
