"""GPU: the ONE-launch stochastic step for small batches (B_sel * k <= 2048, dense uniforms): the selection, accept
test, row choice and offset scans run as the persistent sampler's prologue (csrc/stream.cu fused_select), each CTA
ranking the cells of its own rows against every key.

Bar: bit-identical to the two-launch step (select1_kernel + its epilogue, then persist_stream_kernel — itself pinned
to the oracle) and to the C oracle: windows, win_offsets, PolicyStats, accepted lengths, emitted tokens, row mass,
compaction offsets and the token stream — on adversarial selections (ties, -0.0, quantised scores, ragged rows),
capacity edge cases, emission caps, request shards (row0 > 0) and the logits form.  All calls through the C ABI.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2502_15197_b200 import _native as N
from paper_2502_15197_b200 import ops
from paper_2502_15197_b200.synthetic import make_batch, make_logit_batch, selection_instance

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _np(t):
    return t.detach().cpu().numpy()


class _Out:
    def __init__(self, Bsel, B, k):
        z = lambda n, dt=torch.int32: torch.zeros(n, dtype=dt, device=DEV)  # noqa: E731
        self.windows, self.woff = z(Bsel), z(Bsel + 1)
        self.acc, self.tok, self.mass = z(B), z(B), z(B, torch.float64)
        self.offs, self.toks = z(B + 1), z(max(1, B * (k + 1)))
        self.stats, self.status = z(4, torch.int64), ops.new_status(DEV)

    def results(self):
        n = int(self.offs[-1])
        return {"windows": _np(self.windows), "win_offsets": _np(self.woff), "stats": _np(self.stats)[:3],
                "accepted": _np(self.acc), "out_tok": _np(self.tok), "mass": _np(self.mass).view(np.uint64),
                "offsets": _np(self.offs), "tokens": _np(self.toks)[:n]}


def _run(conf, ln, Bsel, k, C, row0, B, p, q, d, u_acc, u_res, V, cap, fused):
    """fused: tetris_step_stochastic_f32 (one launch when eligible); else its two halves (select1 + epilogue, then the
    plain persistent sampler)."""
    lib, s = N.load(), torch.cuda.current_stream().cuda_stream
    o = _Out(Bsel, B, k)
    ws = ops.Workspace(DEV, N.OP_ALL, Bsel, k, V)
    cp = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    if fused:
        rc = lib.tetris_step_stochastic_f32(
            conf.data_ptr(), cp(ln), Bsel, k, C, row0, B, p.data_ptr(), q.data_ptr(), d.data_ptr(), u_acc.data_ptr(),
            0, u_res.data_ptr(), cp(cap), V, o.windows.data_ptr(), o.woff.data_ptr(), o.acc.data_ptr(),
            o.tok.data_ptr(), o.mass.data_ptr(), o.offs.data_ptr(), o.toks.data_ptr(), o.stats.data_ptr(),
            o.status.data_ptr(), ws.ptr, ws.nbytes, s)
        assert rc == N.OK, lib.tetris_last_error()
    else:
        rc = lib.tetris_select_accept_f32(
            conf.data_ptr(), cp(ln), Bsel, k, C, row0, B, p.data_ptr(), q.data_ptr(), d.data_ptr(), u_acc.data_ptr(),
            0, cp(cap), V, o.windows.data_ptr(), o.woff.data_ptr(), o.acc.data_ptr(), o.offs.data_ptr(),
            o.toks.data_ptr(), o.stats.data_ptr(), o.status.data_ptr(), ws.ptr, ws.nbytes, s)
        assert rc == N.OK, lib.tetris_last_error()
        rc = lib.tetris_resample_f32(p.data_ptr(), q.data_ptr(), u_res.data_ptr(), B, k, V, d.data_ptr(),
                                     o.acc.data_ptr(), o.offs.data_ptr(), o.tok.data_ptr(), o.mass.data_ptr(),
                                     o.toks.data_ptr(), o.status.data_ptr(), ws.ptr, ws.nbytes, s)
        assert rc == N.OK, lib.tetris_last_error()
    torch.cuda.synchronize()
    return o


def _check(B, k, V, C, seed, *, conf=None, lengths=None, cap=False, world=1, rank=0):
    bt = make_batch(B, k, V, seed=seed)
    if conf is None:
        conf, lengths = bt.conf, bt.lengths
    Bsel = B * world
    if world > 1:  # the other shards' scores around this rank's rows
        others = [make_batch(B, k, 8, seed=seed + 1000 + r).conf for r in range(world)]
        others[rank] = conf
        conf = torch.cat(others).contiguous()
        lengths = None if lengths is None else torch.cat([lengths] * world).contiguous()
    g = torch.Generator(DEV).manual_seed(seed + 7)
    capt = torch.randint(0, k + 3, (B,), dtype=torch.int32, device=DEV, generator=g) if cap else None
    args = (conf, lengths, Bsel, k, C, rank * B, B, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res, V, capt)
    one = _run(*args, fused=True)
    two = _run(*args, fused=False)
    ops.raise_for_status(one.status)
    r1, r2 = one.results(), two.results()
    for name in r1:
        assert np.array_equal(r1[name], r2[name]), f"{name}: one-launch step differs from the two-launch step"
    # and the oracle, stage by stage
    w_ref, _, st_ref = O.select(_np(conf), C, None if lengths is None else _np(lengths))
    assert np.array_equal(r1["windows"], w_ref)
    assert list(r1["stats"]) == list(st_ref[:3])
    assert np.array_equal(r1["win_offsets"], np.concatenate([[0], np.cumsum(w_ref)]))
    wl = w_ref[rank * B:(rank + 1) * B]
    acc_ref, tok_ref, mass_ref = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), wl, _np(bt.u_acc),
                                                     _np(bt.u_res), None, nthreads=8)
    assert np.array_equal(r1["accepted"], acc_ref)
    assert np.array_equal(r1["out_tok"], tok_ref)
    assert np.array_equal(r1["mass"], mass_ref.view(np.uint64))
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None if capt is None else _np(capt))
    assert np.array_equal(r1["offsets"], off_ref)
    assert np.array_equal(r1["tokens"], toks_ref)


@pytest.mark.parametrize("B,k,V,C", [(256, 8, 32000, 1024), (16, 5, 32000, 48), (1, 1, 8, 1), (2048, 1, 1024, 700),
                                     (128, 16, 8200, 999), (37, 11, 4096, 200), (200, 10, 128256, 1500)])
def test_one_launch_matches_two_launch_and_oracle(B, k, V, C):
    _check(B, k, V, C, seed=B * 31 + k)


@pytest.mark.parametrize("C", [0, 1, 255, 1024, 2047, 2048, 5000])
def test_capacity_edges(C):
    _check(256, 8, 8192, C, seed=C + 3)


@pytest.mark.parametrize("kind", ["quantized", "ties", "zeros", "ragged"])
def test_adversarial_selection(kind):
    conf, ln = selection_instance(256, 8, kind, seed=11)
    for C in (1, 256, 1023, 2047):
        _check(256, 8, 8192, C, seed=5, conf=conf.contiguous(), lengths=ln.contiguous())


def test_emission_cap():
    _check(256, 8, 32000, 1024, seed=9, cap=True)


@pytest.mark.parametrize("world,rank", [(2, 1), (4, 0), (4, 3)])
def test_request_shard(world, rank):
    """rank r of W: the selection over the W * B gathered rows, verification over this rank's rows only"""
    _check(64, 8, 8192, 300 * world, seed=world * 10 + rank, world=world, rank=rank)


def test_repeated_launches_and_graph_replay():
    """the workspace counters the fused prologue uses are left at zero: many launches in a row (and in a CUDA graph)
    give the same results as the first"""
    B, k, V, C = 256, 8, 32000, 1024
    sets = [make_batch(B, k, V, seed=s) for s in (1, 2)]
    step = ops.TetrisStep(B, k, V, C)
    assert step.fused and step.launches_per_step == 1
    ref = []
    for bt in sets:
        step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
        torch.cuda.synchronize()
        ref.append((step.accepted.clone(), step.out_tok.clone(), step.tokens.clone(), step.windows.clone()))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(4):
                for bt in sets:
                    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(5):
        step.accepted.zero_()
        g.replay()
    torch.cuda.synchronize()
    a, t, tk, w = ref[1]
    assert torch.equal(step.accepted, a) and torch.equal(step.out_tok, t) and torch.equal(step.windows, w)
    assert torch.equal(step.tokens[: int(step.offsets[-1])], tk[: int(step.offsets[-1])])
    for bt, (a, t, tk, w) in zip(sets, ref):  # eager again after the graph: counters still clean
        step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
        torch.cuda.synchronize()
        assert torch.equal(step.accepted, a) and torch.equal(step.out_tok, t)


def test_bad_scores_flagged():
    B, k, V, C = 16, 4, 1024, 20
    bt = make_batch(B, k, V, seed=3)
    conf = bt.conf.clone()
    conf[3, 1] = 1.5  # AcceptanceMatrix rejects probabilities outside [0, 1] (accept_model.py:55-59)
    step = ops.TetrisStep(B, k, V, C)
    step.run(conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    with pytest.raises(ValueError):
        ops.raise_for_status(step.status)


def test_logits_one_launch():
    B, k, V, C = 256, 8, 32000, 1024
    lb = make_logit_batch(B, k, V, seed=5, ragged=True)
    step = ops.TetrisStep(B, k, V, C)
    assert step.fused
    step.run_logits(lb.conf, lb.lengths, lb.zp, lb.lse_p, lb.zq, lb.lse_q, lb.d, lb.u_acc, lb.u_res)
    p = ops.probs_from_logits(lb.zp, lb.lse_p)
    q = ops.probs_from_logits(lb.zq, lb.lse_q)
    s32 = ops.TetrisStep(B, k, V, C)
    s32.run(lb.conf, lb.lengths, p, q, lb.d, lb.u_acc, lb.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    for name in ("windows_all", "win_offsets", "stats", "accepted", "out_tok", "offsets", "mass"):
        a, b = getattr(s32, name), getattr(step, name)
        assert torch.equal(a.view(torch.int64) if a.dtype == torch.float64 else a,
                           b.view(torch.int64) if b.dtype == torch.float64 else b), name
    n = int(step.offsets[-1])
    assert torch.equal(s32.tokens[:n], step.tokens[:n])
    w_ref, _, _ = O.select(_np(lb.conf), C, _np(lb.lengths))
    assert np.array_equal(_np(step.windows_all), w_ref)


# ---------------------------------------------------------------------------------------------------------------
# the one-launch GREEDY step (persist_greedy_kernel<FUSED>): the selection as the argmax stream's prologue while row 0
# of every request streams; against the stage-by-stage path (tetris_select_f64 + tetris_verify_greedy_compact_f32)
# and the oracle
def _greedy_step(conf, ln, Bsel, k, C, row0, B, p, d, V, cap):
    lib, s = N.load(), torch.cuda.current_stream().cuda_stream
    o = _Out(Bsel, B, k)
    ws = ops.Workspace(DEV, N.OP_ALL, Bsel, k, V)
    cp = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    rc = lib.tetris_step_greedy_f32(conf.data_ptr(), cp(ln), Bsel, k, C, row0, B, p.data_ptr(), d.data_ptr(), cp(cap),
                                    V, o.windows.data_ptr(), o.woff.data_ptr(), o.acc.data_ptr(), o.tok.data_ptr(),
                                    o.offs.data_ptr(), o.toks.data_ptr(), o.stats.data_ptr(), o.status.data_ptr(),
                                    ws.ptr, ws.nbytes, s)
    assert rc == N.OK, lib.tetris_last_error()
    torch.cuda.synchronize()
    return o, ws


def _check_greedy(B, k, V, C, seed, *, conf=None, lengths=None, cap=False, world=1, rank=0, repeat=1):
    bt = make_batch(B, k, V, seed=seed, mode="greedy")
    if conf is None:
        conf, lengths = bt.conf, bt.lengths
    Bsel = B * world
    if world > 1:
        others = [make_batch(B, k, 8, seed=seed + 1000 + r).conf for r in range(world)]
        others[rank] = conf
        conf = torch.cat(others).contiguous()
        lengths = None if lengths is None else torch.cat([lengths] * world).contiguous()
    g = torch.Generator(DEV).manual_seed(seed + 7)
    capt = torch.randint(0, k + 3, (B,), dtype=torch.int32, device=DEV, generator=g) if cap else None
    o, ws = _greedy_step(conf, lengths, Bsel, k, C, rank * B, B, bt.p, bt.d, V, capt)
    lib = N.load()
    for _ in range(repeat - 1):  # the same workspace again: ready words / keys / counters left clean
        rc = lib.tetris_step_greedy_f32(conf.data_ptr(), None if lengths is None else lengths.data_ptr(), Bsel, k, C,
                                        rank * B, B, bt.p.data_ptr(), bt.d.data_ptr(),
                                        None if capt is None else capt.data_ptr(), V, o.windows.data_ptr(),
                                        o.woff.data_ptr(), o.acc.data_ptr(), o.tok.data_ptr(), o.offs.data_ptr(),
                                        o.toks.data_ptr(), o.stats.data_ptr(), o.status.data_ptr(), ws.ptr, ws.nbytes,
                                        torch.cuda.current_stream().cuda_stream)
        assert rc == N.OK
    torch.cuda.synchronize()
    ops.raise_for_status(o.status)
    r = o.results()
    w_ref, _, st_ref = O.select(_np(conf), C, None if lengths is None else _np(lengths))
    assert np.array_equal(r["windows"], w_ref)
    assert list(r["stats"]) == list(st_ref[:3])
    assert np.array_equal(r["win_offsets"], np.concatenate([[0], np.cumsum(w_ref)]))
    wl = w_ref[rank * B:(rank + 1) * B]
    acc_ref, tok_ref = O.verify_greedy(_np(bt.p), _np(bt.d), wl, nthreads=8)
    assert np.array_equal(r["accepted"], acc_ref)
    assert np.array_equal(r["out_tok"], tok_ref)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None if capt is None else _np(capt))
    assert np.array_equal(r["offsets"], off_ref)
    assert np.array_equal(r["tokens"], toks_ref)


@pytest.mark.parametrize("B,k,V,C", [(16, 5, 32000, 48), (256, 8, 32000, 1024), (1, 1, 8, 1), (37, 11, 4096, 200),
                                     (2048, 1, 1024, 700), (100, 20, 8200, 900), (128, 16, 128256, 999)])
def test_greedy_one_launch_parity(B, k, V, C):
    _check_greedy(B, k, V, C, seed=B * 7 + k)


@pytest.mark.parametrize("C", [0, 1, 79, 80, 500])
def test_greedy_capacity_edges_and_cap(C):
    _check_greedy(16, 5, 32000, C, seed=C, cap=True)


@pytest.mark.parametrize("kind", ["quantized", "ties", "zeros", "ragged"])
def test_greedy_adversarial_selection(kind):
    conf, ln = selection_instance(256, 8, kind, seed=13)
    _check_greedy(256, 8, 8192, 1000, seed=3, conf=conf.contiguous(), lengths=ln.contiguous())


def test_greedy_shard_and_repeats():
    _check_greedy(64, 8, 8192, 1200, seed=4, world=4, rank=2)
    _check_greedy(64, 8, 8192, 300, seed=5, repeat=4)


def test_greedy_step_launch_count():
    step = ops.TetrisStep(16, 5, 32000, 48, mode="greedy")
    assert step.launches_per_step == 1


@pytest.mark.parametrize("mode", ["stochastic", "greedy"])
@pytest.mark.parametrize("B", [2500, 4096, 5000])
def test_k0_large_batches(mode, B):
    """k = 0 (nothing drafted) gives every batch 0 cells: the one-launch path still holds at most 4096 rows (its scans
    keep 8 rows per thread); larger batches take the two-launch step.  Either way every request emits its bonus
    token, as the oracle says."""
    k, V, C = 0, 8192, 10
    bt = make_batch(B, k, V, seed=B, mode=mode)
    step = ops.TetrisStep(B, k, V, C, mode=mode)
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    ops.raise_for_status(step.status)
    w_ref = np.zeros(B, np.int32)
    if mode == "stochastic":
        acc_ref, tok_ref, _ = O.verify_stochastic(_np(bt.p), _np(bt.q), _np(bt.d), w_ref, _np(bt.u_acc),
                                                  _np(bt.u_res), nthreads=8)
    else:
        acc_ref, tok_ref = O.verify_greedy(_np(bt.p), _np(bt.d), w_ref, nthreads=8)
    off_ref, toks_ref = O.compact(acc_ref, tok_ref, _np(bt.d), None)
    assert np.array_equal(_np(step.windows), w_ref) and np.array_equal(_np(step.out_tok), tok_ref)
    assert np.array_equal(_np(step.offsets), off_ref) and np.array_equal(_np(step.tokens)[: off_ref[-1]], toks_ref)
