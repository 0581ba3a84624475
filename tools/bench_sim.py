"""f1 timing: the reference simulator's run_step (tetris_sched from baseline/_ref, draft phase
excluded) against GpuSimulator.step on the same draft rows and random streams, at a serving-size batch.

Runs the REFERENCE for S steps recording each step's draft-phase rows, then replays them through GpuSimulator (both
PolicyStats modes) and checks every step's windows / accepted / credited / completions against the reference's
StepOutcome.  Prints one JSON line.  usage: python tools/bench_sim.py [B k extra steps]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

B, k, extra, S = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (1024, 8, 8, 30)


def main():
    import tetris_sched.sim_engine as E
    from tetris_sched.accept_model import MixSource, SurrogateConfig

    cfg = E.SimConfig(batch_size=B, k=k, capacity=B * k, seed=5, extra=extra, policy="tetris",
                      acceptance=MixSource(0.95, 0.4, 0.5), surrogate=SurrogateConfig(),
                      target_length=E.UniformLength(16, 256), steps=S)
    cfg.validate()
    streams = [np.random.default_rng(s) for s in np.random.SeedSequence(cfg.seed).spawn(4)]
    lengths = [cfg.target_length.sample(streams[0]) for _ in range(B + 64 * S + 4096)]
    uniforms = streams[3].random(S * cfg.capacity + 16)
    K = k + extra
    state = E.init_state(cfg)
    rec, draft_s = [], [0.0]
    real_draft = E.draft_phase

    def recording_draft(st, cf):
        t0 = time.perf_counter()
        truth, surrogate = real_draft(st, cf)
        draft_s[0] += time.perf_counter() - t0
        tm, sm = np.zeros((B, K)), np.zeros((B, K))
        for i, (tr, sr) in enumerate(zip(truth.rows, surrogate.rows)):
            tm[i, :len(tr)] = tr
            sm[i, :len(sr)] = sr
        rec.append((tm, sm, [len(r) for r in truth.rows]))
        return truth, surrogate

    E.draft_phase = recording_draft
    outs = []
    t0 = time.perf_counter()
    for _ in range(S):
        outs.append(E.run_step(state, cfg))
    ref_s = time.perf_counter() - t0 - draft_s[0]  # draft phase excluded (the caller's part on the GPU path too)
    E.draft_phase = real_draft

    import torch

    from paper_2502_15197_b200.sim_engine import GpuSimulator

    res = {}
    for exact in (True, False):
        sim = GpuSimulator(B, k, cfg.capacity, extra=extra, policy="tetris", uniforms=uniforms, lengths=lengths,
                           device="cuda", exact_stats=exact)
        ok = True
        times = []
        for i, (tm, sm, depths) in enumerate(rec):
            ok &= list(sim.depths()) == depths
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            out = sim.step(tm, sm)
            times.append(time.perf_counter() - t1)
            o = outs[i]
            ok &= (out.windows == tuple(o.windows) and out.accepted == tuple(o.accepted)
                   and out.credited == tuple(o.credited) and out.completions == tuple(o.completions)
                   and out.expected_accepted == o.expected_accepted)
            if exact:
                st = o.stats
                ok &= (out.stats.extracts, out.stats.inserts, out.stats.peak_queue, out.stats.comparisons) == (
                    st.extracts, st.inserts, st.peak_queue, st.comparisons)
        med = float(np.median(times[3:])) if len(times) > 4 else float(np.median(times))
        res["exact_stats" if exact else "closed_form_stats"] = {"ms_per_step": med * 1e3, "matches_reference": ok}
    line = {"what": "GpuSimulator.step vs tetris_sched run_step (draft phase excluded)", "B": B, "k": k,
            "extra": extra, "capacity": cfg.capacity, "steps": S,
            "reference_ms_per_step": ref_s / S * 1e3, "gpu": res,
            "speedup_closed_form": ref_s / S / (res["closed_form_stats"]["ms_per_step"] / 1e3)}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
