"""GPU: the native request-sharded entry points (csrc/dist.cu, tetris_dist_*) at world sizes 2, 4 and 8 on ONE B200.

NCCL cannot form a multi-rank communicator on one device, so the library is pointed ($TETRIS_NCCL_LIB) at an
in-process stand-in (tests/fake_nccl/fake_nccl.cu) whose ncclAllGather is a rendezvous of the W rank threads plus
device-to-device copies ordered by events.  Each rank is a host thread with its own inputs, outputs and workspace,
and calls the library exactly as a multi-GPU serving process would (all ranks enqueue on one stream, so that their
persistent kernels do not share the device's SMs at once, which W processes on W GPUs never do): every rank's
gathered windows must equal the single-device selection over all W*B rows (the CPU oracle's), and each rank's
accepted lengths, emitted tokens and compacted stream the oracle's for its own rows — for the stochastic step (fp32
and logits) and the greedy step."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _build_shim(out_dir: Path) -> Path:
    so = out_dir / "libfake_nccl.so"
    r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                        "-Xcompiler", "-fPIC", "-o", str(so), str(ROOT / "tests" / "fake_nccl" / "fake_nccl.cu")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return so


def _worker(shim: str) -> list:
    os.environ["TETRIS_NCCL_LIB"] = shim  # before the library's first NCCL use (resolved once)
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    try:
        import ctypes as C
        import threading

        import numpy as np
        import torch

        import oracle as O
        from paper_2502_15197_b200 import _native as N
        from paper_2502_15197_b200 import ops
        from paper_2502_15197_b200.synthetic import make_batch, make_logit_batch

        torch.cuda.set_device(0)
        lib = N.load()
        fk = C.CDLL(shim)
        fk.fake_nccl_world_create.restype = C.c_void_p
        fk.fake_nccl_world_create.argtypes = [C.c_int]
        fk.fake_nccl_comm_create.restype = C.c_void_p
        fk.fake_nccl_comm_create.argtypes = [C.c_void_p, C.c_int]
        np_ = lambda t: t.detach().cpu().numpy()  # noqa: E731
        fails = []
        for W, B, k, V, C_, mode, logits in ((2, 300, 8, 8192, 2400, "stochastic", False),
                                             (4, 256, 8, 32000, 4000, "stochastic", False),
                                             (2, 1024, 16, 16384, 20000, "stochastic", False),
                                             (2, 128, 8, 8192, 1000, "stochastic", True),
                                             (4, 16, 5, 32000, 200, "greedy", False),
                                             # SURVEY 8e's determinism check: W = 8 at B = 4096 in total
                                             (8, 512, 16, 4096, 16384, "stochastic", False)):
            world = fk.fake_nccl_world_create(W)
            comms = [fk.fake_nccl_comm_create(world, r) for r in range(W)]
            if logits:
                bts = [make_logit_batch(B, k, V, seed=70 + r, ragged=True) for r in range(W)]
            else:
                bts = [make_batch(B, k, V, mode=mode, seed=70 + r, ragged=True) for r in range(W)]
            steps = [ops.TetrisStep(B, k, V, C_, mode=mode, shard=(W, r)) for r in range(W)]
            # ONE stream for all ranks: their persistent kernels then run one after another (W grids of one CTA per
            # SM on one GPU could otherwise be co-scheduled partially and wait on each other's missing CTAs); the
            # collective itself still needs every rank thread inside it at once
            torch.cuda.synchronize()  # the inputs were made on the default stream; the ranks run on their own
            shared = torch.cuda.Stream()
            streams = [shared] * W
            rcs = [None] * W

            def rank(r):
                torch.cuda.set_device(0)
                st, bt, s = steps[r], bts[r], streams[r].cuda_stream
                common = (st.conf_all.data_ptr(), st.len_all.data_ptr(), st.windows_all.data_ptr(),
                          st.win_offsets.data_ptr(), st.accepted.data_ptr(), st.out_tok.data_ptr())
                if logits:
                    rcs[r] = lib.tetris_dist_step_stochastic_bf16(
                        bt.conf.data_ptr(), bt.lengths.data_ptr(), B, k, C_, bt.zp.data_ptr(), bt.lse_p.data_ptr(),
                        bt.zq.data_ptr(), bt.lse_q.data_ptr(), bt.d.data_ptr(), bt.u_acc.data_ptr(),
                        bt.u_res.data_ptr(), None, V, comms[r], *common, st.mass.data_ptr(), st.offsets.data_ptr(),
                        st.tokens.data_ptr(), st.stats.data_ptr(), st.status.data_ptr(), st.ws.ptr, st.ws.nbytes, s)
                elif mode == "stochastic":
                    rcs[r] = lib.tetris_dist_step_stochastic_f32(
                        bt.conf.data_ptr(), bt.lengths.data_ptr(), B, k, C_, bt.p.data_ptr(), bt.q.data_ptr(),
                        bt.d.data_ptr(), bt.u_acc.data_ptr(), bt.u_res.data_ptr(), None, V, comms[r], *common,
                        st.mass.data_ptr(), st.offsets.data_ptr(), st.tokens.data_ptr(), st.stats.data_ptr(),
                        st.status.data_ptr(), st.ws.ptr, st.ws.nbytes, s)
                else:
                    rcs[r] = lib.tetris_dist_step_greedy_f32(
                        bt.conf.data_ptr(), bt.lengths.data_ptr(), B, k, C_, bt.p.data_ptr(), bt.d.data_ptr(), None,
                        V, comms[r], *common, st.offsets.data_ptr(), st.tokens.data_ptr(), st.stats.data_ptr(),
                        st.status.data_ptr(), st.ws.ptr, st.ws.nbytes, s)
                streams[r].synchronize()

            th = [threading.Thread(target=rank, args=(r,)) for r in range(W)]
            for t in th:
                t.start()
            for t in th:
                t.join(120)
            tag = f"W={W} B={B} k={k} V={V} {mode}{' logits' if logits else ''}"
            if any(rc != N.OK for rc in rcs):
                fails.append(f"{tag}: rc {rcs} {lib.tetris_last_error()}")
                continue
            conf_all = np.concatenate([np_(bt.conf) for bt in bts])
            len_all = np.concatenate([np_(bt.lengths) for bt in bts])
            w_ref, _, _ = O.select(conf_all, C_, len_all)
            for r in range(W):
                st, bt = steps[r], bts[r]
                ops.raise_for_status(st.status, tag)
                if not np.array_equal(np_(st.windows_all), w_ref):
                    fails.append(f"{tag} rank {r}: windows")
                    continue
                wl = w_ref[r * B:(r + 1) * B]
                if logits:
                    p = O.probs_from_logits_bf16(np_(bt.zp.view(torch.int16)).view(np.uint16), np_(bt.lse_p))
                    q = O.probs_from_logits_bf16(np_(bt.zq.view(torch.int16)).view(np.uint16), np_(bt.lse_q))
                    acc, tok, _ = O.verify_stochastic(p, q, np_(bt.d), wl, np_(bt.u_acc), np_(bt.u_res), nthreads=8)
                elif mode == "stochastic":
                    acc, tok, _ = O.verify_stochastic(np_(bt.p), np_(bt.q), np_(bt.d), wl, np_(bt.u_acc),
                                                      np_(bt.u_res), nthreads=8)
                else:
                    acc, tok = O.verify_greedy(np_(bt.p), np_(bt.d), wl, nthreads=8)
                off, toks = O.compact(acc, tok, np_(bt.d))
                ok = (np.array_equal(np_(st.accepted), acc) and np.array_equal(np_(st.out_tok), tok)
                      and np.array_equal(np_(st.offsets), off) and np.array_equal(np_(st.tokens)[: off[-1]], toks))
                if not ok:
                    fails.append(f"{tag} rank {r}: verification")
        return fails
    except Exception:  # pragma: no cover - reported on stdout
        import traceback

        return [traceback.format_exc()]


def test_native_sharded_steps_at_world_2_4_8(tmp_path):
    # a fresh interpreter (the NCCL library is resolved once per process), bounded by a timeout so that a
    # rendezvous that never completes fails the test instead of hanging the suite
    shim = _build_shim(tmp_path)
    r = subprocess.run([sys.executable, __file__, str(shim)], capture_output=True, text=True, timeout=400, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res == [], res


if __name__ == "__main__":
    print(json.dumps(_worker(sys.argv[1])), flush=True)
    os._exit(0)  # the fake worlds' events and threads need no orderly teardown
