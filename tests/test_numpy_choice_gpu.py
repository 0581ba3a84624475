"""Full-vocabulary agreement of the PRODUCT sampler with the reference's own sampling arithmetic (numpy).

The reference samples with `Generator.choice(V, p=...)` (accept_model.py:364, :368): a sequential fp64 cumsum,
normalised by its last entry, searched with searchsorted(..., 'right'); the residual's probabilities come from
residual_distribution's `clip(p - q, 0) / pairwise sum` (accept_model.py:316-327).  A sequential cumsum cannot be
parallelised bit-exactly, so the GPU follows the fixed fp64 reduction tree of include/tetris_b200.h (bit-exact against
the C oracle, tests/test_gpu_parity.py); here the same product path (TetrisStep at cfg3: select + speculative
persistent sampler) is compared with numpy's arithmetic on > 10^6 (row, u) draws at V = 128256, residual and bonus rows
both.  Every disagreement must be a last-bit boundary case: u within 1e-12 of the numpy CDF step between the two
indices.  The count is printed (run with -s) and bounded.
"""
import numpy as np
import pytest
import torch

import reference_port as RP
from paper_2502_15197_b200 import ops
from paper_2502_15197_b200.synthetic import make_batch

pytestmark = pytest.mark.gpu


def test_product_sampler_vs_numpy_choice_cfg3_1M_draws():
    B, k, V, C = 1024, 16, 128256, 8192
    rounds = 1000  # 1000 x 1024 = 1,024,000 draws
    bt = make_batch(B, k, V, seed=2024, device="cuda")
    step = ops.TetrisStep(B, k, V, C, mode="stochastic", device="cuda")
    assert step.uses_spec
    g = torch.Generator(device="cuda")
    g.manual_seed(99)
    U = torch.rand(rounds, B, generator=g, device="cuda", dtype=torch.float64)
    toks = torch.empty(rounds, B, dtype=torch.int32, device="cuda")
    u_res = torch.empty(B, dtype=torch.float64, device="cuda")
    acc0 = None
    for i in range(rounds):
        u_res.copy_(U[i])
        step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, u_res)
        toks[i].copy_(step.out_tok)
        if i == 0:
            acc0 = step.accepted.clone()
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    assert torch.equal(step.accepted, acc0)  # u_acc is fixed: the same row is sampled every round
    acc = step.accepted.long()
    w = step.windows.long()
    resid = acc < w
    ar = torch.arange(B, device="cuda")
    P = bt.p[ar, torch.where(resid, acc, w)].cpu().numpy()
    Q = bt.q[ar, acc.clamp(max=k - 1)].cpu().numpy()
    Uh, T = U.cpu().numpy(), toks.cpu().numpy()
    resid = resid.cpu().numpy()
    mism = {"residual": 0, "bonus": 0}
    draws = {"residual": 0, "bonus": 0}
    worst = 0.0
    for b in range(B):
        kind = "residual" if resid[b] else "bonus"
        cdf = RP.numpy_cdf(P[b], Q[b] if resid[b] else None)
        ref = RP.numpy_choice(cdf, Uh[:, b])
        bad = np.nonzero(ref != T[:, b])[0]
        draws[kind] += rounds
        mism[kind] += len(bad)
        for r in bad:
            lo = min(int(ref[r]), int(T[r, b]))
            hi = max(int(ref[r]), int(T[r, b]))
            # the two indices straddle one CDF step (zero-width steps between them allowed) and u sits on it
            assert np.all(cdf[lo:hi] == cdf[lo]), (b, r, lo, hi)
            gap = abs(float(cdf[lo]) - float(Uh[r, b]))
            worst = max(worst, gap)
            assert gap < 1e-12, f"request {b} round {r}: GPU {T[r, b]} vs numpy {ref[r]}, |u - cdf| = {gap:.3e}"
    total = sum(draws.values())
    n_bad = sum(mism.values())
    print(f"\nnumpy_mismatch: {n_bad} of {total} draws (residual {mism['residual']}/{draws['residual']}, "
          f"bonus {mism['bonus']}/{draws['bonus']}); worst |u - cdf step| among them {worst:.3e}")
    assert total >= 1_000_000 and draws["residual"] > 0 and draws["bonus"] > 0
    assert n_bad <= total * 1e-5
