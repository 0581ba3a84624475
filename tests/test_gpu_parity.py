"""GPU parity: every CUDA stage against the CPU oracle (oracle/tetris_oracle.c) on identical seeded inputs.

Bar: bit-exact windows / stats / cum bits / accepted lengths / emitted tokens / compacted streams; fp64 residual
values within the stated tolerance.  All calls go through the C ABI (paper_2502_15197_b200._native).
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2502_15197_b200 import _native as N
from paper_2502_15197_b200 import ops
from paper_2502_15197_b200.synthetic import make_batch, selection_instance

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _np(t):
    return t.detach().cpu().numpy()


def _check_select(alpha, lengths, C, vals_are_cum=False):
    a = alpha.to(DEV).contiguous()
    ln = None if lengths is None else lengths.to(DEV).contiguous()
    res = ops.select(a, C, ln, vals_are_cum=vals_are_cum, want_cum=True)
    w_ref, cum_ref, st_ref = O.select(_np(a), C, None if ln is None else _np(ln), vals_are_cum=vals_are_cum)
    w = _np(res.windows)
    assert np.array_equal(w, w_ref), f"windows differ at rows {np.nonzero(w != w_ref)[0][:10]}"
    st = _np(res.stats)
    assert st[0] == st_ref[0] and st[1] == st_ref[1] and st[2] == st_ref[2], (st, st_ref)
    off = _np(res.win_offsets)
    assert off[0] == 0 and np.array_equal(np.diff(off), w)
    L = np.full(a.shape[0], a.shape[1]) if ln is None else _np(ln)
    cum = _np(res.cum)
    mask = np.arange(a.shape[1])[None, :] < L[:, None]
    assert np.array_equal(cum[mask].view(np.uint64), cum_ref[mask].view(np.uint64)), "cum bits differ"
    ops.raise_for_status(res.status)
    return res


@pytest.mark.parametrize("seed", range(40))
def test_select_random_small(seed):
    rng = np.random.default_rng(seed)
    B = int(rng.integers(1, 40))
    k = int(rng.integers(1, 9))
    a = torch.from_numpy(rng.random((B, k)))
    ln = torch.from_numpy(rng.integers(1, k + 1, B).astype(np.int32))
    for C in (0, 1, int(rng.integers(0, B * k + 3)), B * k, B * k + 5):
        _check_select(a, ln, C)


@pytest.mark.parametrize("kind", ["quantized", "ties", "zeros", "ragged", "random"])
@pytest.mark.parametrize("B,k", [(16, 5), (256, 8), (1024, 16), (3000, 7)])
def test_select_adversarial(kind, B, k):
    a, ln = selection_instance(B, k, kind, seed=B + k)
    for C in (1, B, B * k // 2, B * k - 1):
        _check_select(a, ln, C)


@pytest.mark.parametrize("B,k,C", [(16, 5, 48), (256, 8, 1024), (1024, 16, 8192), (16384, 16, 131072)]
                         + [(4096, 16, c) for c in (4096, 8192, 16384, 32768, 65536)])
def test_select_configs(B, k, C):
    batch_conf = torch.rand(B, k, dtype=torch.float64, generator=torch.Generator().manual_seed(B * 7 + C))
    _check_select(batch_conf ** 0.25, None, C)


@pytest.mark.parametrize("kind", ["quantized", "ties", "random", "ragged"])
@pytest.mark.parametrize("B,k", [(300, 20), (2000, 40), (70, 255), (12000, 17)])
def test_select_shared_memory_path(kind, B, k):
    """k > 16 (or more than 16384 rows) takes the shared-memory key path instead of the register path."""
    a, ln = selection_instance(B, k, kind, seed=B * k)
    for C in (1, B, B * k // 3, B * k - 1):
        _check_select(a, ln, C)


def test_select_given_cum_nonmonotone():
    """select_tetris over arbitrary Candidate.cum lists (heap merge == top-C over the prefix-min envelope)."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        B, k = int(rng.integers(1, 30)), int(rng.integers(1, 7))
        cum = np.round(rng.random((B, k)) * 8) / 8  # many ties, non-monotone rows
        ln = rng.integers(0, k + 1, B).astype(np.int32)
        for C in (1, int(rng.integers(0, B * k + 1)), B * k):
            _check_select(torch.from_numpy(cum), torch.from_numpy(ln), C, vals_are_cum=True)


def test_heap_stats_exact_comparisons():
    rng = np.random.default_rng(11)
    for _ in range(30):
        B, k = int(rng.integers(1, 64)), int(rng.integers(1, 10))
        a = torch.from_numpy(rng.random((B, k))).to(DEV)
        C = int(rng.integers(0, B * k + 2))
        res = ops.select(a, C, want_cum=True)
        st = _np(ops.heap_stats(res.cum, C))
        _, _, st_ref = O.select(_np(a), C)
        assert np.array_equal(st, st_ref), (st, st_ref)


def test_select_negative_capacity():
    with pytest.raises(ValueError):
        ops.select(torch.rand(2, 2, dtype=torch.float64, device=DEV), -1)


def test_select_bad_alpha_flagged():
    a = torch.tensor([[0.5, 1.5]], dtype=torch.float64, device=DEV)
    res = ops.select(a, 1)
    with pytest.raises(ValueError):
        ops.raise_for_status(res.status)


# ---------------------------------------------------------------------------------------------------------------
def _stochastic_parity(B, k, V, C, seed, ragged=False, packed=False):
    bt = make_batch(B, k, V, seed=seed, ragged=ragged)
    sel = ops.select(bt.conf, C, bt.lengths)
    if packed:
        n = int(sel.win_offsets[-1].item())
        u_acc = torch.rand(max(n, 1), dtype=torch.float64, device=DEV, generator=torch.Generator(DEV).manual_seed(seed))
        res = ops.verify_stochastic(bt.p, bt.q, bt.d, sel.windows, u_acc, bt.u_res, sel.win_offsets, want_mass=True)
        woff = _np(sel.win_offsets)
    else:
        u_acc = bt.u_acc
        res = ops.verify_stochastic(bt.p, bt.q, bt.d, sel.windows, u_acc, bt.u_res, want_mass=True)
        woff = None
    ops.raise_for_status(res.status)
    acc_ref, tok_ref, mass_ref = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), _np(sel.windows), _np(u_acc),
                                                     _np(bt.u_res), woff, nthreads=8)
    acc, tok, mass = _np(res.accepted), _np(res.out_tok), _np(res.mass)
    assert np.array_equal(acc, acc_ref), f"accepted differ at {np.nonzero(acc != acc_ref)[0][:10]}"
    assert np.array_equal(tok, tok_ref), f"tokens differ at {np.nonzero(tok != tok_ref)[0][:10]}"
    assert np.array_equal(mass.view(np.uint64), mass_ref.view(np.uint64)), "mass bits differ"
    off, toks = ops.compact(res.accepted, res.out_tok, bt.d)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d))
    assert np.array_equal(_np(off), off_ref)
    assert np.array_equal(_np(toks)[: off_ref[-1]], toks_ref)
    return acc, _np(sel.windows)


@pytest.mark.parametrize("B,k,V,C,seed", [(16, 5, 32000, 48, 0), (256, 8, 32000, 1024, 1), (64, 8, 1000, 300, 2),
                                          (33, 3, 8200, 40, 3), (7, 2, 13, 9, 4), (128, 16, 128256, 1024, 5)])
def test_stochastic_parity(B, k, V, C, seed):
    acc, w = _stochastic_parity(B, k, V, C, seed)
    assert (acc <= w).all()


def test_stochastic_parity_ragged_packed():
    _stochastic_parity(100, 6, 4096, 333, 7, ragged=True, packed=True)


def test_greedy_parity():
    for (B, k, V, C, seed) in [(16, 5, 32000, 48, 0), (64, 4, 1003, 100, 1), (200, 8, 32000, 900, 2)]:
        bt = make_batch(B, k, V, seed=seed, mode="greedy")
        sel = ops.select(bt.conf, C, bt.lengths)
        res = ops.verify_greedy(bt.p, bt.d, sel.windows)
        ops.raise_for_status(res.status)
        acc_ref, tok_ref = O.verify_greedy(_np(bt.p), _np(bt.d), _np(sel.windows), nthreads=8)
        assert np.array_equal(_np(res.accepted), acc_ref)
        assert np.array_equal(_np(res.out_tok), tok_ref)


def test_greedy_ties_and_nan():
    B, k, V = 4, 2, 300
    p = torch.zeros(B, k + 1, V, dtype=torch.float32)
    p[0, :, 5] = 1.0
    p[0, :, 7] = 1.0          # tie -> first index 5
    p[1, 0, 9] = float("nan")  # NaN ranks highest
    p[1, 0, 3] = 2.0
    p[2, :, 299] = 0.5
    p[3, 1, 0] = -0.0
    d = torch.tensor([[5, 5], [9, 1], [299, 299], [0, 1]], dtype=torch.int32)
    w = torch.tensor([2, 2, 1, 2], dtype=torch.int32)
    res = ops.verify_greedy(p.to(DEV), d.to(DEV), w.to(DEV))
    acc_ref, tok_ref = O.verify_greedy(p.numpy(), d.numpy(), w.numpy())
    assert np.array_equal(_np(res.accepted), acc_ref)
    assert np.array_equal(_np(res.out_tok), tok_ref)


def test_sample_rows_and_residual_f64():
    rng = np.random.default_rng(3)
    for V in (2, 3, 8, 100, 8191, 8192, 8193, 40000):
        R = 5
        ps = rng.dirichlet(np.ones(V), size=R)
        pt = rng.dirichlet(np.ones(V), size=R)
        u = rng.random(R)
        rows = torch.arange(R, dtype=torch.int64, device=DEV)
        idx, mass, st = ops.sample_rows(torch.from_numpy(pt).to(DEV), rows, torch.from_numpy(u).to(DEV),
                                        q=torch.from_numpy(ps).to(DEV), q_row=rows)
        ops.raise_for_status(st)
        for r in range(R):
            i_ref, m_ref = O.sample(pt[r], u[r], q=ps[r])
            assert int(idx[r]) == i_ref and float(mass[r]) == m_ref
        out, mass2, st = ops.residual(torch.from_numpy(ps).to(DEV), torch.from_numpy(pt).to(DEV))
        ops.raise_for_status(st)
        for r in range(R):
            ref, m_ref, rc = O.residual(ps[r], pt[r])
            assert rc == 0 and float(mass2[r]) == m_ref
            assert np.array_equal(_np(out[r]), ref)
            # against the reference's own formula (pairwise np.sum mass): fp64 tolerance
            diff = np.clip(pt[r] - ps[r], 0.0, None)
            np.testing.assert_allclose(_np(out[r]), diff / diff.sum(), rtol=1e-12, atol=1e-15)


def test_residual_degenerate():
    p = torch.tensor([[0.3, 0.7]], dtype=torch.float64, device=DEV)
    _, _, st = ops.residual(p, p.clone())
    from paper_2502_15197_b200.errors import DegenerateResidualError

    with pytest.raises(DegenerateResidualError):
        ops.raise_for_status(st)


def test_verify_matrix_parity():
    rng = np.random.default_rng(9)
    B, k = 500, 9
    alpha = rng.random((B, k))
    w = rng.integers(0, k + 1, B).astype(np.int32)
    off = np.zeros(B + 1, np.int32)
    off[1:] = np.cumsum(w)
    u = rng.random(max(1, off[-1]))
    acc = ops.verify_matrix(torch.from_numpy(alpha).to(DEV), torch.from_numpy(w).to(DEV),
                            torch.from_numpy(off).to(DEV), torch.from_numpy(u).to(DEV))
    assert np.array_equal(_np(acc), O.verify_matrix(alpha, w, u))


def test_expected_accepted_parity():
    rng = np.random.default_rng(4)
    alpha = rng.random((300, 7))
    w = rng.integers(0, 8, 300).astype(np.int32)
    v = ops.expected_accepted(torch.from_numpy(alpha).to(DEV), torch.from_numpy(w).to(DEV))
    assert float(v) == O.expected_accepted(alpha, w)


def test_compact_cap():
    rng = np.random.default_rng(1)
    B, k = 300, 6
    acc = rng.integers(0, k + 1, B).astype(np.int32)
    tok = rng.integers(0, 100, B).astype(np.int32)
    d = rng.integers(0, 100, (B, k)).astype(np.int32)
    cap = rng.integers(1, k + 3, B).astype(np.int32)
    off, toks = ops.compact(*(torch.from_numpy(x).to(DEV) for x in (acc, tok, d, cap)))
    off_ref, toks_ref = O.compact(acc, tok, d, cap)
    assert np.array_equal(_np(off), off_ref)
    assert np.array_equal(_np(toks)[: off_ref[-1]], toks_ref)


def test_step_graph_capture_matches_eager():
    B, k, V, C = 64, 8, 32000, 256
    bt = make_batch(B, k, V, seed=21)
    step = ops.TetrisStep(B, k, V, C)
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ref = (step.accepted.clone(), step.out_tok.clone(), step.tokens.clone())
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        step.accepted.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(step.accepted, ref[0]) and torch.equal(step.out_tok, ref[1])
    assert torch.equal(step.tokens, ref[2])


# ---------------------------------------------------------------------------------------------------------------
# the fused two-launch step (select+accept+offsets, persistent TMA sampler) == the stage-by-stage oracle
def _fused_vs_oracle(B, k, V, C, seed, ragged=False, packed=False, cap=False):
    bt = make_batch(B, k, V, seed=seed, ragged=ragged)
    step = ops.TetrisStep(B, k, V, C, u_layout="packed" if packed else "dense")
    g = torch.Generator(DEV).manual_seed(seed + 1)
    u_acc = torch.rand(B * k, dtype=torch.float64, device=DEV, generator=g) if packed else bt.u_acc
    capt = torch.randint(1, k + 3, (B,), dtype=torch.int32, device=DEV, generator=g) if cap else None
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, u_acc, bt.u_res, cap=capt)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    w_ref, _, st_ref = O.select(_np(bt.conf), C, _np(bt.lengths))
    assert np.array_equal(_np(step.windows), w_ref)
    assert list(_np(step.stats)[:3]) == list(st_ref[:3])
    woff = np.concatenate([[0], np.cumsum(w_ref)]).astype(np.int32)
    acc_ref, tok_ref, mass_ref = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), w_ref, _np(u_acc),
                                                     _np(bt.u_res), woff if packed else None, nthreads=8)
    assert np.array_equal(_np(step.accepted), acc_ref)
    assert np.array_equal(_np(step.out_tok), tok_ref)
    assert np.array_equal(_np(step.mass).view(np.uint64), mass_ref.view(np.uint64))
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None if capt is None else _np(capt))
    assert np.array_equal(_np(step.offsets), off_ref)
    assert np.array_equal(_np(step.tokens)[: off_ref[-1]], toks_ref)


@pytest.mark.parametrize("B,k,V,C,seed", [(16, 5, 32000, 48, 0), (256, 8, 32000, 1024, 1), (300, 7, 8200, 900, 2),
                                          (1, 1, 8, 1, 3), (64, 16, 128256, 512, 4), (2000, 4, 1024, 3000, 5)])
def test_fused_step_parity(B, k, V, C, seed):
    _fused_vs_oracle(B, k, V, C, seed)


def test_fused_step_ragged_packed_cap():
    _fused_vs_oracle(200, 6, 4096, 700, 11, ragged=True, packed=True, cap=True)
    _fused_vs_oracle(200, 6, 4096, 700, 12, ragged=True, packed=False, cap=True)


def test_fused_step_full_cfg3_bit_exact():
    """BASELINE cfg3 at full size (B=1024, k=16, C=8192, V=128256): every request's accepted length, emitted token
    and row mass against the oracle.  Only the rows the oracle needs are copied to the host."""
    B, k, V, C = 1024, 16, 128256, 8192
    bt = make_batch(B, k, V, seed=42)
    step = ops.TetrisStep(B, k, V, C)
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    w_ref, _, _ = O.select(_np(bt.conf), C)
    assert np.array_equal(_np(step.windows), w_ref)
    # accept test from gathered values (torch gather, independent of the kernels)
    d = bt.d.long()
    m = bt.p[:, :k].gather(2, d.unsqueeze(-1)).squeeze(-1).double().cpu().numpy()
    s = bt.q.gather(2, d.unsqueeze(-1)).squeeze(-1).double().cpu().numpy()
    u = _np(bt.u_acc)
    acc_ref = np.zeros(B, np.int64)
    for b in range(B):
        a = w_ref[b]
        for j in range(w_ref[b]):
            if not (s[b, j] <= m[b, j] or u[b, j] < m[b, j] / s[b, j]):
                a = j
                break
        acc_ref[b] = a
    assert np.array_equal(_np(step.accepted), acc_ref)
    ures = _np(bt.u_res)
    tok = _np(step.out_tok)
    mass = _np(step.mass)
    for b0 in range(0, B, 128):
        bs = np.arange(b0, min(B, b0 + 128))
        a = acc_ref[bs]
        rej = a < w_ref[bs]
        prow = bt.p[torch.from_numpy(bs).to(DEV), torch.from_numpy(np.where(rej, a, w_ref[bs])).to(DEV)].cpu().numpy()
        qrow = bt.q[torch.from_numpy(bs).to(DEV), torch.from_numpy(np.minimum(a, k - 1)).to(DEV)].cpu().numpy()
        for i, b in enumerate(bs):
            t, mm = O.sample(prow[i], ures[b], q=qrow[i] if rej[i] else None)
            assert tok[b] == t and mass[b] == mm, b


# ---------------------------------------------------------------------------------------------------------------
# the request-sharded step of rank r in a world of W (what TetrisStep(group=...) launches after the all-gather),
# simulated on one GPU: the selection runs over the gathered W*B rows with the global capacity, the verification
# tensors cover only this rank's rows
@pytest.mark.parametrize("W,B,k,V,C,rank", [(2, 512, 16, 8192, 8192, 1), (4, 1024, 16, 4096, 32768, 3),
                                             (8, 1024, 16, 2048, 65536, 5), (2, 300, 7, 4096, 2000, 0),
                                             # >= 4096 streamed chunks: the speculative sampler behind the single-CTA
                                             # selector (W=2) and behind the grid selector (W=8)
                                             (2, 512, 16, 65536, 8192, 1), (8, 1024, 4, 32768, 16384, 6)])
def test_sharded_step_matches_global_selection(W, B, k, V, C, rank):
    shards = [make_batch(B, k, V, seed=100 + r) for r in range(W)]
    conf_all = torch.cat([s.conf for s in shards]).contiguous()
    len_all = torch.cat([s.lengths for s in shards]).contiguous()
    bt = shards[rank]
    Bg = W * B
    lib = N.load()
    dev = bt.p.device
    windows = torch.zeros(Bg, dtype=torch.int32, device=dev)
    woff = torch.zeros(Bg + 1, dtype=torch.int32, device=dev)
    acc = torch.zeros(B, dtype=torch.int32, device=dev)
    tok = torch.zeros(B, dtype=torch.int32, device=dev)
    mass = torch.zeros(B, dtype=torch.float64, device=dev)
    offs = torch.zeros(B + 1, dtype=torch.int32, device=dev)
    toks = torch.zeros(B * (k + 1), dtype=torch.int32, device=dev)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    status = ops.new_status(dev)
    ws = ops.Workspace(dev, N.OP_ALL, Bg, k, V)
    rc = lib.tetris_step_stochastic_f32(
        conf_all.data_ptr(), len_all.data_ptr(), Bg, k, C, rank * B, B, bt.p.data_ptr(), bt.q.data_ptr(),
        bt.d.data_ptr(), bt.u_acc.data_ptr(), 0, bt.u_res.data_ptr(), None, V, windows.data_ptr(), woff.data_ptr(),
        acc.data_ptr(), tok.data_ptr(), mass.data_ptr(), offs.data_ptr(), toks.data_ptr(), stats.data_ptr(),
        status.data_ptr(), ws.ptr, ws.nbytes, torch.cuda.current_stream().cuda_stream)
    assert rc == N.OK, lib.tetris_last_error()
    torch.cuda.synchronize()
    ops.raise_for_status(status)
    w_ref, _, st_ref = O.select(_np(conf_all), C, _np(len_all))
    assert np.array_equal(_np(windows), w_ref)
    assert list(_np(stats)[:3]) == list(st_ref[:3])
    wl = w_ref[rank * B:(rank + 1) * B]
    acc_ref, tok_ref, mass_ref = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), wl, _np(bt.u_acc),
                                                     _np(bt.u_res), None, nthreads=8)
    assert np.array_equal(_np(acc), acc_ref)
    assert np.array_equal(_np(tok), tok_ref)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None)
    assert np.array_equal(_np(offs), off_ref)
    assert np.array_equal(_np(toks)[: off_ref[-1]], toks_ref)


def _adversarial_rows(V, rng):
    """fp32 rows the sampler must treat exactly like the oracle: sparse spikes, exact zeros, subnormals, p == q ties,
    tiny residual mass, huge dynamic range."""
    rows = []
    sub = np.float32(1e-40)  # subnormal
    a = np.zeros(V, np.float32); a[rng.integers(0, V, 3)] = [0.5, 0.25, 0.25]; rows.append(a)
    b = np.full(V, sub, np.float32); b[V // 2] = 1.0; rows.append(b)
    c = rng.random(V).astype(np.float32) * np.float32(1e-30); c[::7] = 0; rows.append(c)
    d = (rng.random(V) ** 8).astype(np.float32); rows.append(d)
    e = np.zeros(V, np.float32); e[-1] = 1e-38; e[0] = 3e-39; rows.append(e)
    return rows


def test_sampler_adversarial_rows_f32():
    rng = np.random.default_rng(77)
    for V in (8, 8192, 8200, 32000, 128256):
        P = _adversarial_rows(V, rng)
        Q = [np.roll(x, 1) for x in P]  # residual partners; row 0 vs its shift, ties where both are 0
        Q[3] = P[3].copy(); Q[3][::3] = 0  # p == q on two thirds of the row: tiny residual
        R = len(P)
        p = torch.from_numpy(np.stack(P)).to(DEV)
        q = torch.from_numpy(np.stack(Q)).to(DEV)
        rows = torch.arange(R, dtype=torch.int64, device=DEV)
        for u_val in (0.0, 0.37, 1.0 - 2.0 ** -53):
            u = torch.full((R,), u_val, dtype=torch.float64, device=DEV)
            for residual in (False, True):
                idx, mass, st = ops.sample_rows(p, rows, u, q=q if residual else None,
                                                q_row=rows if residual else None)
                torch.cuda.synchronize()
                for r in range(R):
                    i_ref, m_ref = O.sample(P[r], u_val, q=Q[r] if residual else None)
                    assert float(mass[r]) == m_ref, (V, r, residual)
                    if m_ref > 0:
                        assert int(idx[r]) == i_ref, (V, r, u_val, residual)


# ---------------------------------------------------------------------------------------------------------------
# the speculative sampler (tetris_resample_spec_f32): the rows of requests rejected at their first drafted token are
# streamed before the selection completes; results identical to the plain sampler and the oracle, including the
# requests it streams for nothing (window 0), empty rows, out-of-vocabulary first tokens, repeated calls
@pytest.mark.parametrize("B,k,V,C,seed,ragged", [(64, 4, 8200, 10, 1, True), (300, 6, 4096, 40, 2, True),
                                                  (1024, 16, 32000, 8192, 3, False), (2048, 3, 1024, 3000, 4, True),
                                                  (4096, 2, 1024, 5000, 6, True),
                                                  (5, 2, 8, 3, 5, False)])
def test_spec_sampler_matches_oracle(B, k, V, C, seed, ragged):
    bt = make_batch(B, k, V, seed=seed, ragged=ragged)
    if ragged:
        bt.lengths[::7] = 0  # empty rows: nothing drafted, never speculative
    bt.d[::5, 0] = V + 3     # out-of-vocabulary first token: rejected at 0
    lib = N.load()
    dev = bt.p.device
    outs = {}
    for variant in ("spec", "plain"):
        step = ops.TetrisStep(B, k, V, C)
        for it in range(3):
            step.status.zero_()
            rc = lib.tetris_select_accept_f32(
                bt.conf.data_ptr(), bt.lengths.data_ptr(), B, k, C, 0, B, bt.p.data_ptr(), bt.q.data_ptr(),
                bt.d.data_ptr(), bt.u_acc.data_ptr(), 0, None, V, step.windows_all.data_ptr(),
                step.win_offsets.data_ptr(), step.accepted.data_ptr(), step.offsets.data_ptr(), step.tokens.data_ptr(),
                step.stats.data_ptr(), step.status.data_ptr(), step.ws.ptr, step.ws.nbytes,
                torch.cuda.current_stream().cuda_stream)
            assert rc == N.OK, lib.tetris_last_error()
            if variant == "spec":
                rc = lib.tetris_resample_spec_f32(
                    bt.p.data_ptr(), bt.q.data_ptr(), bt.u_res.data_ptr(), bt.u_acc.data_ptr(), bt.lengths.data_ptr(),
                    B, k, V, bt.d.data_ptr(), step.accepted.data_ptr(), step.offsets.data_ptr(),
                    step.out_tok.data_ptr(), step.mass.data_ptr(), step.tokens.data_ptr(), step.status.data_ptr(),
                    step.ws.ptr, step.ws.nbytes, torch.cuda.current_stream().cuda_stream)
            else:
                rc = lib.tetris_resample_f32(
                    bt.p.data_ptr(), bt.q.data_ptr(), bt.u_res.data_ptr(), B, k, V, bt.d.data_ptr(),
                    step.accepted.data_ptr(), step.offsets.data_ptr(), step.out_tok.data_ptr(), step.mass.data_ptr(),
                    step.tokens.data_ptr(), step.status.data_ptr(), step.ws.ptr, step.ws.nbytes,
                    torch.cuda.current_stream().cuda_stream)
            assert rc == N.OK, lib.tetris_last_error()
            torch.cuda.synchronize()
            outs.setdefault(variant, []).append(tuple(_np(x).copy() for x in (
                step.windows, step.accepted, step.out_tok, step.mass, step.offsets, step.tokens, step.status)))
    for o in outs["spec"] + outs["plain"][1:]:
        for x, y in zip(o, outs["plain"][0]):
            assert np.array_equal(x.view(np.uint8), y.view(np.uint8))
    w, acc, tok, mass, off, toks, st = outs["spec"][0]
    w_ref, _, _ = O.select(_np(bt.conf), C, _np(bt.lengths))
    assert np.array_equal(w, w_ref)
    acc_ref, tok_ref, mass_ref = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), w_ref, _np(bt.u_acc),
                                                     _np(bt.u_res), None, nthreads=8)
    assert np.array_equal(acc, acc_ref) and np.array_equal(tok, tok_ref)
    assert np.array_equal(mass.view(np.uint64), mass_ref.view(np.uint64))
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None)
    assert np.array_equal(off, off_ref) and np.array_equal(toks[: off_ref[-1]], toks_ref)
    if B >= 64:
        assert (w == 0).any() or C >= B  # the window-0 path is exercised where the capacity is tight


@pytest.mark.parametrize("seed", range(8))
def test_spec_sampler_random_shapes(seed):
    """Seeded random shapes through the speculative sampler explicitly (tight and loose capacities, ragged depths,
    V with a partial last chunk), against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 700))
    k = int(rng.integers(1, 12))
    V = int(rng.choice([8, 1000, 8192, 8200, 20000]))
    V -= V % 8
    C = int(rng.integers(0, B * k + 2))
    bt = make_batch(B, k, V, seed=seed, ragged=bool(seed % 2))
    step = ops.TetrisStep(B, k, V, C)
    lib = N.load()
    s = torch.cuda.current_stream().cuda_stream
    assert lib.tetris_select_accept_f32(
        bt.conf.data_ptr(), bt.lengths.data_ptr(), B, k, C, 0, B, bt.p.data_ptr(), bt.q.data_ptr(), bt.d.data_ptr(),
        bt.u_acc.data_ptr(), 0, None, V, step.windows_all.data_ptr(), step.win_offsets.data_ptr(),
        step.accepted.data_ptr(), step.offsets.data_ptr(), step.tokens.data_ptr(), step.stats.data_ptr(),
        step.status.data_ptr(), step.ws.ptr, step.ws.nbytes, s) == N.OK
    assert lib.tetris_resample_spec_f32(
        bt.p.data_ptr(), bt.q.data_ptr(), bt.u_res.data_ptr(), bt.u_acc.data_ptr(), bt.lengths.data_ptr(), B, k, V,
        bt.d.data_ptr(), step.accepted.data_ptr(), step.offsets.data_ptr(), step.out_tok.data_ptr(),
        step.mass.data_ptr(), step.tokens.data_ptr(), step.status.data_ptr(), step.ws.ptr, step.ws.nbytes, s) == N.OK
    torch.cuda.synchronize()
    w_ref, _, _ = O.select(_np(bt.conf), C, _np(bt.lengths))
    assert np.array_equal(_np(step.windows), w_ref)
    acc_ref, tok_ref, mass_ref = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), w_ref, _np(bt.u_acc),
                                                     _np(bt.u_res), None, nthreads=8)
    assert np.array_equal(_np(step.accepted), acc_ref) and np.array_equal(_np(step.out_tok), tok_ref)
    assert np.array_equal(_np(step.mass).view(np.uint64), mass_ref.view(np.uint64))
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None)
    assert np.array_equal(_np(step.offsets), off_ref)
    assert np.array_equal(_np(step.tokens)[: off_ref[-1]], toks_ref)


@pytest.mark.parametrize("V", [1003, 13, 8191])
def test_step_stochastic_any_vocabulary(V):
    """V % 8 != 0: TetrisStep runs the stage-by-stage kernels (the TMA sampler needs 32-byte rows); same results as
    the oracle."""
    B, k, C = 90, 5, 200
    bt = make_batch(B, k, V, seed=V, ragged=True)
    step = ops.TetrisStep(B, k, V, C)
    assert step.launches_per_step == 3
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    w_ref, _, _ = O.select(_np(bt.conf), C, _np(bt.lengths))
    acc_ref, tok_ref, mass_ref = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), w_ref, _np(bt.u_acc),
                                                     _np(bt.u_res), None, nthreads=8)
    assert np.array_equal(_np(step.accepted), acc_ref) and np.array_equal(_np(step.out_tok), tok_ref)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None)
    assert np.array_equal(_np(step.offsets), off_ref)
    assert np.array_equal(_np(step.tokens)[: off_ref[-1]], toks_ref)



@pytest.mark.parametrize("B,k", [(4096, 16), (1000, 40), (20000, 3)])
def test_cluster_selector_without_workspace(B, k):
    """tetris_select_f64 with no workspace runs the cluster/DSMEM select_kernel for B*k > 16384 (register path for
    k <= 16, shared-memory path above); bit-exact against the oracle like the workspace selectors."""
    rng = np.random.default_rng(B + k)
    a = torch.from_numpy(rng.random((B, k)) ** 0.3).to(DEV)
    ln = torch.from_numpy(rng.integers(1, k + 1, B).astype(np.int32)).to(DEV)
    for C in (1, B, B * k // 3, B * k - 1):
        w = torch.empty(B, dtype=torch.int32, device=DEV)
        off = torch.empty(B + 1, dtype=torch.int32, device=DEV)
        cum = torch.zeros(B, k, dtype=torch.float64, device=DEV)
        st = torch.zeros(4, dtype=torch.int64, device=DEV)
        status = ops.new_status(DEV)
        N.call("tetris_select_f64", a.data_ptr(), ln.data_ptr(), B, k, C, 0, w.data_ptr(), off.data_ptr(),
               cum.data_ptr(), st.data_ptr(), status.data_ptr(), None, 0, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        ops.raise_for_status(status)
        w_ref, cum_ref, st_ref = O.select(_np(a), C, _np(ln))
        assert np.array_equal(_np(w), w_ref)
        assert list(_np(st)[:3]) == list(st_ref[:3])
        assert np.array_equal(np.diff(_np(off)), w_ref)


def test_misaligned_probabilities_take_the_stage_by_stage_path():
    """A contiguous but not 16-byte aligned p / q view (V % 8 == 0) must not reach the TMA sampler:
    TetrisStep routes it to the stage-by-stage kernels with identical results."""
    B, k, V, C = 32, 4, 4096, 80
    bt = make_batch(B, k, V, seed=4)
    pb = torch.empty(bt.p.numel() + 1, dtype=torch.float32, device=DEV)
    qb = torch.empty(bt.q.numel() + 1, dtype=torch.float32, device=DEV)
    p = pb[1:].view(bt.p.shape)
    q = qb[1:].view(bt.q.shape)
    p.copy_(bt.p)
    q.copy_(bt.q)
    assert p.data_ptr() % 16 and q.data_ptr() % 16 and p.is_contiguous()
    s1 = ops.TetrisStep(B, k, V, C)
    s1.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    s2 = ops.TetrisStep(B, k, V, C)
    s2.run(bt.conf, bt.lengths, p, q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(s2.status)
    assert torch.equal(s1.accepted, s2.accepted) and torch.equal(s1.out_tok, s2.out_tok)
    assert torch.equal(s1.offsets, s2.offsets)


def test_spec_max_requests_follows_the_device():
    from paper_2502_15197_b200 import _native as N2

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert N2.spec_max_requests() == min(4096, 32 * sms)


@pytest.mark.parametrize("kind", ["random", "ties", "ragged"])
@pytest.mark.parametrize("B,k", [(2048, 16), (4096, 16), (1500, 40), (3000, 7)])
def test_select_cluster_kernel_without_workspace(kind, B, k):
    """tetris_select_f64 with NO workspace takes the thread-block-cluster selector (select_kernel, DSMEM histograms)
    for batches above the single-CTA selector's 16384 cells: same windows / stats / cum bits as the oracle."""
    a, ln = selection_instance(B, k, kind, seed=B * k)
    a, ln = a.to(DEV).contiguous(), ln.to(DEV).contiguous()
    for C in (1, B, B * k // 3, B * k - 1):
        windows = torch.zeros(B, dtype=torch.int32, device=DEV)
        offs = torch.zeros(B + 1, dtype=torch.int32, device=DEV)
        cum = torch.zeros(B, k, dtype=torch.float64, device=DEV)
        stats = torch.zeros(4, dtype=torch.int64, device=DEV)
        status = ops.new_status(DEV)
        N.call("tetris_select_f64", a.data_ptr(), ln.data_ptr(), B, k, C, 0, windows.data_ptr(), offs.data_ptr(),
               cum.data_ptr(), stats.data_ptr(), status.data_ptr(), None, 0, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        ops.raise_for_status(status)
        w_ref, cum_ref, st_ref = O.select(_np(a), C, _np(ln))
        assert np.array_equal(_np(windows), w_ref), (kind, B, k, C)
        assert np.array_equal(_np(stats)[:3], st_ref[:3])
        assert np.array_equal(np.diff(_np(offs)), w_ref)
        mask = np.arange(k)[None, :] < _np(ln)[:, None]
        assert np.array_equal(_np(cum)[mask].view(np.uint64), cum_ref[mask].view(np.uint64))


@pytest.mark.parametrize("B,k,V,C", [(64, 4, 16384, 160), (1024, 16, 8192, 8192)])
def test_step_adversarial_rows_through_the_stream_kernel(B, k, V, C):
    """The product sampler (persist_stream_kernel: the fused one-launch step at the small size, the speculative
    two-launch step at the large one) on rows with exact zeros, subnormals, NaN, p == q ties and huge dynamic range
    mixed with ordinary rows: the consumers' integer-widening fast path and their F2F path give the oracle's tokens."""
    bt = make_batch(B, k, V, seed=B + V)
    rng = np.random.default_rng(5)
    p = bt.p.cpu().numpy()
    q = bt.q.cpu().numpy()
    adv = _adversarial_rows(V, rng)
    nan_row = rng.random(V).astype(np.float32)
    nan_row[rng.integers(0, V, 5)] = np.nan
    adv.append(nan_row)
    for b in range(0, B, 3):  # every third request: all its rows adversarial
        for j in range(k + 1):
            p[b, j] = adv[(b + j) % len(adv)]
            if j < k:
                q[b, j] = np.roll(adv[(b + 2 * j + 1) % len(adv)], j + 1)
    pt, qt = torch.from_numpy(p).to(DEV), torch.from_numpy(q).to(DEV)
    step = ops.TetrisStep(B, k, V, C)
    step.run(bt.conf, bt.lengths, pt, qt, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    w_ref, _, _ = O.select(_np(bt.conf), C, _np(bt.lengths))
    acc_ref, tok_ref, _ = O.verify_stochastic(p, q, _np(bt.d), w_ref, _np(bt.u_acc), _np(bt.u_res), nthreads=8)
    assert np.array_equal(_np(step.windows), w_ref)
    assert np.array_equal(_np(step.accepted), acc_ref)
    assert np.array_equal(_np(step.out_tok), tok_ref)


@pytest.mark.parametrize("seed", range(6))
def test_grid_selector_edge_bins(seed):
    """The grid selector's first pass clamps keys outside [2^-127, 1] into its two edge bins (then refines them from
    bit 63): candidate cums above 1, tiny, zero, -0.0 and negative values, with ties, at grid-selector sizes."""
    rng = np.random.default_rng(seed)
    B, k = 4096, 16
    cum = np.sort(rng.random((B, k)), axis=1)[:, ::-1].copy()  # non-increasing rows
    kind = seed % 3
    if kind == 0:    # many scores above 1 (edge bin 0 holds the C-th)
        cum[: B // 2] += rng.integers(1, 4, (B // 2, 1))
    elif kind == 1:  # many tiny / zero / negative scores (edge bin 2047)
        cum[B // 3:] *= 1e-300
        cum[B // 2:, k // 2:] = 0.0
        cum[-B // 8:, -2:] = -np.abs(cum[-B // 8:, -2:]) - 1.0
        cum[B // 2: B // 2 + 50, -1] = -0.0
    else:            # quantised ties spanning both edges
        cum = np.round(cum * 8) / 8 * rng.choice([1e-200, 1.0, 3.0], (B, 1))
    cum = np.minimum.accumulate(cum, axis=1)  # keep rows non-increasing (the candidate lists' envelope)
    lens = rng.integers(1, k + 1, B).astype(np.int32)
    for C in (1, 777, B * k // 4, B * k // 2, B * k - 3):
        _check_select(torch.from_numpy(cum), torch.from_numpy(lens), C, vals_are_cum=True)
