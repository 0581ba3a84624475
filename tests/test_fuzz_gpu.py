"""GPU: randomised shapes through the product entry points against the C oracle (bit-exact).

Every draw picks B, k, V (including V % 8 != 0 and single-chunk rows), C (0, tiny, B*k and above), ragged depths,
the verification mode and — for the stochastic step — the input form (fp32 probabilities or bf16 logits + lse, the
latter materialised through the logits contract for the oracle), and sometimes an emission cap.  The dispatch between
the one-launch, two-launch, speculative, grid-selector and stage-by-stage paths is the library's own, so the draws
sweep across all of them."""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2502_15197_b200 import ops
from paper_2502_15197_b200.synthetic import make_batch, make_logit_batch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


def _bits(z: torch.Tensor) -> np.ndarray:
    return z.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


# TETRIS_FUZZ_DRAWS raises the draw count for a long one-off run (the suite's default stays at 80)
@pytest.mark.parametrize("seed", range(int(os.environ.get("TETRIS_FUZZ_DRAWS", "80"))))
def test_random_shapes_match_the_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.choice([1, 3, 16, 37, 130, 300, 700, 1100, 2100]))
    k = int(rng.integers(1, 17))
    V = int(rng.choice([8, 64, 1000, 1003, 8192, 8200, 16384, 32000]))
    mode = "greedy" if rng.random() < 0.35 else "stochastic"
    logits = mode == "stochastic" and V % 8 == 0 and rng.random() < 0.4
    cells = B * k
    C = int(rng.choice([0, 1, B, cells // 2, cells, cells + 7]))
    ragged = bool(rng.random() < 0.6)
    cap = torch.from_numpy(rng.integers(0, k + 2, B).astype(np.int32)).cuda() if rng.random() < 0.3 else None
    step = ops.TetrisStep(B, k, V, C, mode=mode)
    if logits:
        lb = make_logit_batch(B, k, V, seed=seed, ragged=ragged)
        step.run_logits(lb.conf, lb.lengths, lb.zp, lb.lse_p, lb.zq, lb.lse_q, lb.d, lb.u_acc, lb.u_res, cap=cap)
        p = O.probs_from_logits_bf16(_bits(lb.zp), _np(lb.lse_p))
        q = O.probs_from_logits_bf16(_bits(lb.zq), _np(lb.lse_q))
        conf, lengths, d, u_acc, u_res = lb.conf, lb.lengths, lb.d, lb.u_acc, lb.u_res
    else:
        bt = make_batch(B, k, V, seed=seed, mode=mode, ragged=ragged)
        step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res, cap=cap)
        p, q = _np(bt.p), (_np(bt.q) if mode == "stochastic" else None)
        conf, lengths, d, u_acc, u_res = bt.conf, bt.lengths, bt.d, bt.u_acc, bt.u_res
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    w_ref, _, st_ref = O.select(_np(conf), C, _np(lengths))
    assert np.array_equal(_np(step.windows), w_ref), (B, k, V, C, mode, logits)
    assert np.array_equal(_np(step.stats)[:3], st_ref[:3])
    if mode == "stochastic":
        acc_ref, tok_ref, _ = O.verify_stochastic(p, q, _np(d), w_ref, _np(u_acc), _np(u_res), nthreads=8)
    else:
        acc_ref, tok_ref = O.verify_greedy(p, _np(d), w_ref, nthreads=8)
    assert np.array_equal(_np(step.accepted), acc_ref), (B, k, V, C, mode, logits)
    assert np.array_equal(_np(step.out_tok), tok_ref), (B, k, V, C, mode, logits)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(d), None if cap is None else _np(cap))
    assert np.array_equal(_np(step.offsets), off_ref)
    assert np.array_equal(_np(step.tokens)[: off_ref[-1]], toks_ref)
