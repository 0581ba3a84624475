"""GPU parity of the greedy product path (greedy_rowmap_kernel + persist_greedy_kernel, csrc/greedy.cu) against the CPU
oracle: accepted lengths, emitted tokens and the fused compaction bit-exact, numpy.argmax order on adversarial rows
(NaN, +-inf, -0.0, ties inside and across 8192-element chunks, a partial last chunk), windows 0 / deeper than k,
depths beyond one warp (k > 32), repeated calls on one workspace and CUDA-graph replay.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2502_15197_b200 import _native as N
from paper_2502_15197_b200 import ops
from paper_2502_15197_b200.synthetic import make_batch

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _np(t):
    return t.detach().cpu().numpy()


def _greedy_compact(p, d, w, cap=None):
    """tetris_verify_greedy_compact_f32 through the C ABI."""
    B, k1, V = p.shape
    k = k1 - 1
    acc = torch.full((B,), -7, dtype=torch.int32, device=DEV)
    tok = torch.full((B,), -7, dtype=torch.int32, device=DEV)
    off = torch.full((B + 1,), -7, dtype=torch.int32, device=DEV)
    toks = torch.full((max(1, B * k1),), -7, dtype=torch.int32, device=DEV)
    st = ops.new_status(DEV)
    ws = ops.Workspace(torch.device(DEV), N.OP_VERIFY, B, k, V)
    lib = N.load()
    rc = lib.tetris_verify_greedy_compact_f32(p.data_ptr(), d.data_ptr(), w.data_ptr(),
                                              None if cap is None else cap.data_ptr(), B, k, V, acc.data_ptr(),
                                              tok.data_ptr(), off.data_ptr(), toks.data_ptr(), st.data_ptr(), ws.ptr,
                                              ws.nbytes, torch.cuda.current_stream().cuda_stream)
    assert rc == N.OK, lib.tetris_last_error()
    torch.cuda.synchronize()
    return acc, tok, off, toks, st


def _check(p, d, w, cap=None, expect_status=0):
    acc, tok, off, toks, st = _greedy_compact(p, d, w, cap)
    acc_ref, tok_ref = O.verify_greedy(_np(p), _np(d), _np(w), nthreads=8)
    assert np.array_equal(_np(acc), acc_ref), np.nonzero(_np(acc) != acc_ref)[0][:10]
    assert np.array_equal(_np(tok), tok_ref), np.nonzero(_np(tok) != tok_ref)[0][:10]
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(d), None if cap is None else _np(cap))
    assert np.array_equal(_np(off), off_ref)
    assert np.array_equal(_np(toks)[: off_ref[-1]], toks_ref)
    assert int(st[0]) == expect_status, hex(int(st[0]))
    # the verify-only entry point on the same inputs
    res = ops.verify_greedy(p, d, w)
    torch.cuda.synchronize()
    assert np.array_equal(_np(res.accepted), acc_ref) and np.array_equal(_np(res.out_tok), tok_ref)


@pytest.mark.parametrize("B,k,V,C,seed", [(16, 5, 32000, 48, 0), (200, 8, 32000, 900, 1), (64, 16, 128256, 512, 2),
                                          (3, 40, 8200, 100, 3), (1, 1, 8, 1, 4), (500, 3, 8192, 700, 5)])
def test_greedy_persistent_parity(B, k, V, C, seed):
    bt = make_batch(B, k, V, seed=seed, mode="greedy")
    sel = ops.select(bt.conf, C, bt.lengths)
    g = torch.Generator(DEV).manual_seed(seed)
    cap = torch.randint(0, k + 3, (B,), dtype=torch.int32, device=DEV, generator=g)
    _check(bt.p, bt.d, sel.windows)
    _check(bt.p, bt.d, sel.windows, cap=cap)


def test_greedy_persistent_all_positions_k_beyond_a_warp():
    # k = 40 > 32 lanes, every position drafted as the target's argmax: all accepted, bonus from position w
    B, k, V = 5, 40, 1024
    g = torch.Generator(DEV).manual_seed(9)
    p = torch.rand(B, k + 1, V, dtype=torch.float32, device=DEV, generator=g)
    d = p[:, :k].argmax(-1).to(torch.int32).contiguous()
    w = torch.tensor([40, 33, 32, 31, 0], dtype=torch.int32, device=DEV)
    _check(p, d, w)
    d2 = d.clone()
    d2[0, 35] = (d2[0, 35] + 1) % V  # first mismatch in the second lane group
    d2[1, 32] = (d2[1, 32] + 1) % V
    _check(p, d2, w)


def test_greedy_persistent_adversarial_rows():
    B, k, V = 10, 2, 8200  # two chunks, the second holds 8 elements
    p = torch.zeros(B, k + 1, V, dtype=torch.float32)
    p[0, :, 100] = 1.0
    p[0, :, 8195] = 1.0                       # tie across chunks -> 100
    p[1, 0, 8199] = float("nan")              # NaN in the partial last chunk ranks highest
    p[1, 0, 3] = float("inf")
    p[2, :, 8100] = float("nan")
    p[2, :, 8196] = float("nan")              # first NaN wins, across chunks
    p[3, :, :] = float("-inf")                # all -inf -> index 0
    p[4, :, 0] = -0.0
    p[4, :, 1] = 0.0                          # -0.0 == +0.0 -> index 0 (row otherwise zero)
    p[5, :, :] = -1.0
    p[5, :, 4000] = -0.5
    p[6, :, 8191] = 3.0
    p[6, :, 8192] = 3.0                       # tie at the chunk boundary -> 8191
    p[7, :, 7] = float("inf")
    p[7, :, 9] = float("inf")
    p[8, :, :] = 1e-45                        # subnormal plateau -> index 0
    p[9, 1, 5] = 2.0
    d = torch.tensor([[100, 100], [8199, 0], [8100, 8100], [0, 0], [0, 0], [4000, 4000], [8191, 8191], [7, 9],
                      [0, 1], [0, 5]], dtype=torch.int32)
    w = torch.tensor([2, 2, 2, 2, 2, 2, 2, 2, 2, 0], dtype=torch.int32)
    _check(p.to(DEV), d.to(DEV), w.to(DEV))


def test_greedy_persistent_bad_window_and_token():
    B, k, V = 4, 3, 64
    g = torch.Generator().manual_seed(1)
    p = torch.rand(B, k + 1, V, generator=g)
    d = p[:, :k].argmax(-1).to(torch.int32)
    d[1, 1] = V + 5                           # out of the vocabulary: rejected, flagged
    w = torch.tensor([3, 3, 2, 3], dtype=torch.int32)
    _check(p.to(DEV), d.to(DEV), w.to(DEV), expect_status=N.ST_BAD_TOKEN)
    w_bad = torch.tensor([3, 1, k + 4, -2], dtype=torch.int32)  # clamped to [0, k] and flagged
    d_ok = p[:, :k].argmax(-1).to(torch.int32)
    acc, tok, off, toks, st = _greedy_compact(p.to(DEV), d_ok.to(DEV), w_bad.to(DEV))
    assert int(st[0]) & N.ST_BAD_WINDOW
    acc_ref, tok_ref = O.verify_greedy(p.numpy(), d_ok.numpy(), np.clip(w_bad.numpy(), 0, k))
    assert np.array_equal(_np(acc), acc_ref) and np.array_equal(_np(tok), tok_ref)


def test_greedy_persistent_repeat_and_graph():
    """Counters and the work counter are left at zero: back-to-back calls on one workspace, then graph replays."""
    B, k, V, C = 128, 6, 16384, 400
    bt = make_batch(B, k, V, seed=31, mode="greedy")
    step = ops.TetrisStep(B, k, V, C, mode="greedy")
    outs = []
    for _ in range(3):
        step.run(bt.conf, bt.lengths, bt.p, None, bt.d)
        torch.cuda.synchronize()
        outs.append((step.accepted.clone(), step.out_tok.clone(), step.offsets.clone(), step.tokens.clone()))
    w_ref, _, _ = O.select(_np(bt.conf), C, _np(bt.lengths))
    acc_ref, tok_ref = O.verify_greedy(_np(bt.p), _np(bt.d), w_ref, nthreads=8)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d))
    for a, t, o, s in outs:
        assert np.array_equal(_np(a), acc_ref) and np.array_equal(_np(t), tok_ref)
        assert np.array_equal(_np(o), off_ref) and np.array_equal(_np(s)[: off_ref[-1]], toks_ref)
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            step.run(bt.conf, bt.lengths, bt.p, None, bt.d)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(4):
        step.accepted.zero_()
        step.tokens.zero_()
        gr.replay()
    torch.cuda.synchronize()
    assert np.array_equal(_np(step.accepted), acc_ref) and np.array_equal(_np(step.out_tok), tok_ref)
    assert np.array_equal(_np(step.tokens)[: off_ref[-1]], toks_ref)
    ops.raise_for_status(step.status)


@pytest.mark.parametrize("W,B,k,V,C,rank", [(1, 16, 5, 32000, 48, 0), (1, 1024, 16, 4096, 8192, 0),
                                             (2, 512, 16, 8192, 8192, 1), (4, 1024, 16, 2048, 32768, 3),
                                             (1, 2048, 9, 1024, 9000, 0), (2, 300, 7, 1003, 2000, 1)])
def test_step_greedy_matches_oracle(W, B, k, V, C, rank):
    """tetris_step_greedy_f32 for rank r of W (selection over the gathered W*B rows, verification of the local
    rows): the fused row list (B*W*k <= 16384), the grid selector + row-list kernel (larger), and the stage-by-stage
    fallback (V % 8 != 0)."""
    shards = [make_batch(B, k, V, seed=200 + r, mode="greedy") for r in range(W)]
    conf_all = torch.cat([s.conf for s in shards]).contiguous()
    len_all = torch.cat([s.lengths for s in shards]).contiguous()
    bt = shards[rank]
    Bg = W * B
    lib = N.load()
    dev = bt.p.device
    g = torch.Generator(DEV).manual_seed(rank)
    cap = torch.randint(0, k + 3, (B,), dtype=torch.int32, device=DEV, generator=g)
    windows = torch.zeros(Bg, dtype=torch.int32, device=dev)
    woff = torch.zeros(Bg + 1, dtype=torch.int32, device=dev)
    acc = torch.full((B,), -5, dtype=torch.int32, device=dev)
    tok = torch.full((B,), -5, dtype=torch.int32, device=dev)
    offs = torch.zeros(B + 1, dtype=torch.int32, device=dev)
    toks = torch.zeros(B * (k + 1), dtype=torch.int32, device=dev)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    status = ops.new_status(dev)
    ws = ops.Workspace(dev, N.OP_ALL, Bg, k, V)
    for _ in range(2):  # the second call checks that every counter was left at zero
        rc = lib.tetris_step_greedy_f32(
            conf_all.data_ptr(), len_all.data_ptr(), Bg, k, C, rank * B, B, bt.p.data_ptr(), bt.d.data_ptr(),
            cap.data_ptr(), V, windows.data_ptr(), woff.data_ptr(), acc.data_ptr(), tok.data_ptr(), offs.data_ptr(),
            toks.data_ptr(), stats.data_ptr(), status.data_ptr(), ws.ptr, ws.nbytes,
            torch.cuda.current_stream().cuda_stream)
        assert rc == N.OK, lib.tetris_last_error()
        torch.cuda.synchronize()
        ops.raise_for_status(status)
        w_ref, _, st_ref = O.select(_np(conf_all), C, _np(len_all))
        assert np.array_equal(_np(windows), w_ref)
        assert np.array_equal(_np(woff), np.concatenate([[0], np.cumsum(w_ref)]).astype(np.int32))
        assert list(_np(stats)[:3]) == list(st_ref[:3])
        wl = w_ref[rank * B:(rank + 1) * B]
        acc_ref, tok_ref = O.verify_greedy(_np(bt.p), _np(bt.d), wl, nthreads=8)
        assert np.array_equal(_np(acc), acc_ref) and np.array_equal(_np(tok), tok_ref)
        off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), _np(cap))
        assert np.array_equal(_np(offs), off_ref)
        assert np.array_equal(_np(toks)[: off_ref[-1]], toks_ref)


@pytest.mark.parametrize("seed", range(8))
def test_step_greedy_random_shapes(seed):
    """Seeded random shapes through the fused greedy step (row 0 streamed early, rows 1..w from the selector's row
    list), against the oracle."""
    rng = np.random.default_rng(2000 + seed)
    B = int(rng.integers(1, 600))
    k = int(rng.integers(1, 20))
    V = int(rng.choice([8, 1000, 8192, 8200, 20000]))
    V -= V % 8
    C = int(rng.integers(0, B * k + 2))
    bt = make_batch(B, k, V, seed=seed, mode="greedy", ragged=bool(seed % 2))
    step = ops.TetrisStep(B, k, V, C, mode="greedy")
    step.run(bt.conf, bt.lengths, bt.p, None, bt.d)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    w_ref, _, _ = O.select(_np(bt.conf), C, _np(bt.lengths))
    assert np.array_equal(_np(step.windows), w_ref)
    acc_ref, tok_ref = O.verify_greedy(_np(bt.p), _np(bt.d), w_ref, nthreads=8)
    assert np.array_equal(_np(step.accepted), acc_ref) and np.array_equal(_np(step.out_tok), tok_ref)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None)
    assert np.array_equal(_np(step.offsets), off_ref)
    assert np.array_equal(_np(step.tokens)[: off_ref[-1]], toks_ref)


@pytest.mark.parametrize("mode", ["greedy", "stochastic"])
def test_step_zero_draft_depth(mode):
    """k = 0 (nothing drafted): every window is 0, the emitted token comes from position 0 (the bonus row)."""
    B, k, V, C = 37, 0, 8192, 5
    bt = make_batch(B, k, V, seed=3, mode=mode)
    step = ops.TetrisStep(B, k, V, C, mode=mode)
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    assert int(step.windows.abs().sum()) == 0 and int(step.accepted.abs().sum()) == 0
    if mode == "greedy":
        _, tok_ref = O.verify_greedy(_np(bt.p), _np(bt.d), np.zeros(B, np.int32), nthreads=8)
    else:
        _, tok_ref, _ = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), np.zeros(B, np.int32), _np(bt.u_acc),
                                            _np(bt.u_res), None, nthreads=8)
    assert np.array_equal(_np(step.out_tok), tok_ref)
    assert np.array_equal(_np(step.offsets), np.arange(B + 1, dtype=np.int32))
    assert np.array_equal(_np(step.tokens)[:B], tok_ref)
