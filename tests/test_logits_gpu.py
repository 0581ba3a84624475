"""GPU: the logits form of the stochastic step ("fused bf16 logits -> probs").

The contract (include/tetris_b200.h, "the logits contract"): prob(z, lse) in fp32 with FMA; the C oracle
(oracle_probs_from_logits_bf16, C fmaf) reproduces it bit for bit, and the logits step must equal the fp32 step / the
fp32 oracle applied to those probabilities bit for bit (windows, accepted lengths, tokens, compacted stream, mass).
Tolerance (stated): |prob / exp(x) - 1| <= 1e-6 for x = fp32(z - lse) in [-86, 88]."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2502_15197_b200 import ops
from paper_2502_15197_b200.synthetic import make_logit_batch

pytestmark = pytest.mark.gpu


def _bits(z: torch.Tensor) -> np.ndarray:
    return z.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def test_contract_bits_match_the_oracle_and_exp():
    rng = np.random.default_rng(0)
    R, V = 64, 4099
    zf = (rng.normal(0, 6, (R, V)) * rng.choice([1, 4, 20], (R, 1))).astype(np.float32)
    z = torch.from_numpy(zf).to(torch.bfloat16)
    specials = torch.tensor([float("nan"), float("inf"), -float("inf"), 3e38, -3e38, 0.0, -0.0, 1e-40],
                            dtype=torch.bfloat16)
    z[0, : specials.numel()] = specials
    lse = torch.from_numpy(rng.normal(5, 20, R).astype(np.float32))
    lse[1] = 1e30
    lse[2] = -1e30
    out = ops.probs_from_logits(z.cuda(), lse.cuda()).cpu().numpy()
    ref = O.probs_from_logits_bf16(_bits(z), lse.numpy())
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
    x = z.float().numpy() - lse.numpy()[:, None]  # fp32 RN, as the contract's x (before the row clamp)
    sane = np.ones(R, bool)
    sane[[1, 2]] = False  # |lse| = 1e30: outside the contract's domain (defined bits, not exp)
    m = (x >= -85) & (x <= 87) & sane[:, None]
    rel = np.abs(out[m].astype(np.float64) / np.exp(x[m].astype(np.float64)) - 1)
    assert rel.max() <= 1e-6, rel.max()
    assert np.all(out[sane] > 0) and np.all(np.isfinite(out[sane]))
    # below the clamp every probability reads as ~exp(-86): positive, normal, tiny
    low = (x < -87) & sane[:, None]
    assert np.all(out[low] >= np.float32(1.1754944e-38)) and np.all(out[low] < 1e-36)


@pytest.mark.parametrize("B,k,V,C,ragged", [(16, 5, 32000, 48, False), (256, 8, 32000, 1024, True),
                                            (64, 16, 8200, 300, True), (300, 4, 16384, 700, False)])
def test_logits_step_matches_fp32_step_and_oracle(B, k, V, C, ragged):
    lb = make_logit_batch(B, k, V, seed=B + k, ragged=ragged)
    p = ops.probs_from_logits(lb.zp, lb.lse_p)
    q = ops.probs_from_logits(lb.zq, lb.lse_q)
    s32 = ops.TetrisStep(B, k, V, C)
    s32.run(lb.conf, lb.lengths, p, q, lb.d, lb.u_acc, lb.u_res)
    sbf = ops.TetrisStep(B, k, V, C)
    sbf.run_logits(lb.conf, lb.lengths, lb.zp, lb.lse_p, lb.zq, lb.lse_q, lb.d, lb.u_acc, lb.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(sbf.status)
    for name in ("windows_all", "accepted", "out_tok", "offsets", "mass"):
        a, b = getattr(s32, name), getattr(sbf, name)
        assert torch.equal(a.view(torch.int64) if a.dtype == torch.float64 else a,
                           b.view(torch.int64) if b.dtype == torch.float64 else b), name
    n = int(sbf.offsets[-1])
    assert torch.equal(s32.tokens[:n], sbf.tokens[:n])
    # the oracle on the oracle's own probabilities
    P = O.probs_from_logits_bf16(_bits(lb.zp), lb.lse_p.cpu().numpy())
    Q = O.probs_from_logits_bf16(_bits(lb.zq), lb.lse_q.cpu().numpy())
    w_ref, _, _ = O.select(lb.conf.cpu().numpy(), C, lb.lengths.cpu().numpy())
    acc, tok, mass = O.verify_stochastic(P, Q, lb.d.cpu().numpy(), w_ref, lb.u_acc.cpu().numpy(),
                                         lb.u_res.cpu().numpy(), None, nthreads=8)
    assert np.array_equal(sbf.windows_all.cpu().numpy(), w_ref)
    assert np.array_equal(sbf.accepted.cpu().numpy(), acc)
    assert np.array_equal(sbf.out_tok.cpu().numpy(), tok)


def test_logits_step_cfg3_speculative():
    """cfg3 shape (B=1024, k=16, V=128256): the speculative logits sampler, against the fp32 step on the materialised
    probabilities (bit-exact) and the C oracle on a sample of requests."""
    B, k, V, C = 1024, 16, 128256, 8192
    lb = make_logit_batch(B, k, V, seed=3)
    sbf = ops.TetrisStep(B, k, V, C)
    assert sbf.uses_spec
    for _ in range(2):  # twice: the workspace counters are left at zero
        sbf.run_logits(lb.conf, lb.lengths, lb.zp, lb.lse_p, lb.zq, lb.lse_q, lb.d, lb.u_acc, lb.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(sbf.status)
    p = ops.probs_from_logits(lb.zp, lb.lse_p)
    q = ops.probs_from_logits(lb.zq, lb.lse_q)
    s32 = ops.TetrisStep(B, k, V, C)
    s32.run(lb.conf, lb.lengths, p, q, lb.d, lb.u_acc, lb.u_res)
    torch.cuda.synchronize()
    assert torch.equal(s32.accepted, sbf.accepted) and torch.equal(s32.out_tok, sbf.out_tok)
    assert torch.equal(s32.mass.view(torch.int64), sbf.mass.view(torch.int64))
    assert torch.equal(s32.offsets, sbf.offsets)
    n = 48
    P = O.probs_from_logits_bf16(_bits(lb.zp[:n]), lb.lse_p[:n].cpu().numpy())
    Q = O.probs_from_logits_bf16(_bits(lb.zq[:n]), lb.lse_q[:n].cpu().numpy())
    w = sbf.windows_all.cpu().numpy()[:n]
    acc, tok, _ = O.verify_stochastic(P, Q, lb.d[:n].cpu().numpy(), w, lb.u_acc[:n].cpu().numpy(),
                                      lb.u_res[:n].cpu().numpy(), None, nthreads=8)
    assert np.array_equal(sbf.accepted.cpu().numpy()[:n], acc)
    assert np.array_equal(sbf.out_tok.cpu().numpy()[:n], tok)


def test_logits_step_graph_capture():
    B, k, V, C = 256, 8, 32000, 1024
    lb = make_logit_batch(B, k, V, seed=11)
    st = ops.TetrisStep(B, k, V, C)
    run = lambda: st.run_logits(lb.conf, lb.lengths, lb.zp, lb.lse_p, lb.zq, lb.lse_q, lb.d, lb.u_acc,  # noqa
                                lb.u_res)
    run()
    torch.cuda.synchronize()
    ref = st.out_tok.clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            run()
    torch.cuda.current_stream().wait_stream(s)
    st.out_tok.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(st.out_tok, ref)


@pytest.mark.parametrize("B,k,V,C", [(64, 8, 16384, 200), (200, 5, 8200, 500)])
def test_host_logit_step_matches_device_step(B, k, V, C):
    lb = make_logit_batch(B, k, V, seed=B + k, ragged=True)
    dev = ops.TetrisStep(B, k, V, C)
    dev.run_logits(lb.conf, lb.lengths, lb.zp, lb.lse_p, lb.zq, lb.lse_q, lb.d, lb.u_acc, lb.u_res)
    torch.cuda.synchronize()
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    hs = ops.HostLogitStep(B, k, V, C, pin(lb.zp), pin(lb.lse_p), pin(lb.zq), pin(lb.lse_q))
    small = [pin(t) for t in (lb.conf, lb.lengths, lb.d, lb.u_acc, lb.u_res)]
    for _ in range(2):
        hs.run(*small)
        torch.cuda.synchronize()
        n = int(hs.offsets_host[-1])
        assert np.array_equal(hs.offsets_host.numpy(), dev.offsets.cpu().numpy())
        assert np.array_equal(hs.tokens_host.numpy()[:n], dev.tokens.cpu().numpy()[:n])
        assert np.array_equal(hs.accepted_host.numpy(), dev.accepted.cpu().numpy())
    ops.raise_for_status(hs.step.status)
