"""CPU: the bench's reference arm (oracle/ref_arm.py) -- tetris_sched's own functions composed per step -- agrees
with the C oracle and the port on seeded batches, on one thread and on the process pool."""
import numpy as np
import pytest
import torch

import oracle as O
import ref_arm
import reference_port as RP
from paper_2502_15197_b200.synthetic import make_batch


@pytest.mark.parametrize("mode", ["stochastic", "greedy"])
def test_reference_step_matches_oracle(mode):
    B, k, V, C = 24, 6, 1000, 70
    bt = make_batch(B, k, V, mode=mode, seed=5, device="cpu")
    h = {"p": bt.p.numpy(), "q": bt.q.numpy(), "d": bt.d.numpy(), "conf": bt.conf.numpy(),
         "lengths": bt.lengths.numpy(), "u_acc": bt.u_acc.numpy(), "u_res": bt.u_res.numpy()}
    w_ref, _, _ = O.select(h["conf"], C)
    rs = ref_arm.ReferenceStep(h, C, mode, processes=2).start_pool()
    try:
        _, _, toks1, out1 = rs.run(B, parallel=False)
        _, _, toks2, out2 = rs.run(B, parallel=True)
    finally:
        rs.close()
    assert out1 == out2 and toks1 == toks2 == sum(a + 1 for a, _ in out1)
    assert np.array_equal(np.asarray(ref_arm.select(rs.rows, C)), w_ref)
    if mode == "greedy":
        acc, tok = O.verify_greedy(h["p"], h["d"], w_ref)
    else:
        acc, tok, _ = O.verify_stochastic(h["p"], h["q"], h["d"], w_ref, h["u_acc"], h["u_res"])
    assert [a for a, _ in out1] == list(acc)
    # the emitted token is numpy's choice arithmetic: equal to the fixed-tree contract except at last-bit CDF ties
    assert sum(x == t for (_, x), t in zip(out1, tok)) >= B - 1
    port = [RP.verify_request(h["p"][b], h["q"][b], h["d"][b], w_ref[b], h["u_acc"][b], h["u_res"][b])
            if mode == "stochastic" else RP.verify_request_greedy(h["p"][b], h["d"][b], w_ref[b]) for b in range(B)]
    assert out1 == port


def test_numpy_agreement_counts_mismatches():
    rng = np.random.default_rng(0)
    P = rng.dirichlet(np.ones(50), 6).astype(np.float32)
    Q = rng.dirichlet(np.ones(50), 6).astype(np.float32)
    resid = np.array([True, False, True, False, True, True])
    u = rng.random(6)
    n, ref = ref_arm.numpy_agreement(P, Q, resid, u, np.zeros(6, np.int64))
    assert n == int(np.count_nonzero(ref != 0))
    n2, _ = ref_arm.numpy_agreement(P, Q, resid, u, ref)
    assert n2 == 0
