"""Golden simulator traces for the GPU-resident run_step (paper_2502_15197_b200.sim_engine.GpuSimulator).

Run in the build container (where /root/reference exists):  python tests/golden/make_golden_sim.py
It runs the REFERENCE simulator (tetris_sched 0.1.0, run_step / init_state, sim_engine.py:311-495) read-only and
records, per step, the draft phase's truth and surrogate rows (the inputs the GPU step takes from the caller) and the
StepOutcome fields plus the DSD estimate; and per run the target-length stream and the verify-uniform stream the
reference consumed (numpy PCG64 streams spawned from the seed, sim_engine.py:313).  Arrays are stored as base64 of
their little-endian bytes, so every float is bit-exact.  The GPU box never runs this script; sim.json travels.
"""
from __future__ import annotations

import base64
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "sim.json"


def enc(a, dtype) -> str:
    return base64.b64encode(np.ascontiguousarray(a, dtype=dtype).tobytes()).decode()


def main():
    sys.path.insert(0, str(REF))
    import tetris_sched.sim_engine as E
    from tetris_sched.accept_model import BetaSource, MixSource, SurrogateConfig
    from tetris_sched.trace_io import write_trace

    runs = []
    cases = [
        dict(tag="tetris-mix", batch_size=8, k=4, extra=4, policy="tetris", seed=7,
             acceptance=MixSource(0.95, 0.4, 0.5), target=(10, 40), steps=40),
        dict(tag="tetris-noisy-surrogate", batch_size=8, k=3, extra=5, policy="tetris", seed=11,
             acceptance=BetaSource(4.0, 2.0), surrogate=SurrogateConfig("logit-gaussian", 0.7), target=(5, 30),
             steps=40),
        dict(tag="tetris-beta-b32", batch_size=32, k=4, extra=4, policy="tetris", seed=3,
             acceptance=BetaSource(2.0, 1.0), target=(4, 60), steps=30),
        dict(tag="sd-mix", batch_size=8, k=4, extra=2, policy="sd", seed=5,
             acceptance=MixSource(0.9, 0.3, 0.5), target=(6, 25), steps=40),
        dict(tag="dsd-beta", batch_size=16, k=3, extra=3, policy="dsd", seed=9,
             acceptance=BetaSource(3.0, 1.0, per_row=True), target=(3, 20), steps=40),
    ]
    for c in cases:
        cfg = E.SimConfig(batch_size=c["batch_size"], k=c["k"], capacity=c["batch_size"] * c["k"], seed=c["seed"],
                          extra=c["extra"], policy=c["policy"], acceptance=c["acceptance"],
                          surrogate=c.get("surrogate", SurrogateConfig()),
                          target_length=E.UniformLength(*c["target"]), steps=c["steps"])
        cfg.validate()
        # the streams the reference will consume, re-drawn from identically spawned generators
        streams = [np.random.default_rng(s) for s in np.random.SeedSequence(cfg.seed).spawn(4)]
        lengths = [cfg.target_length.sample(streams[0]) for _ in range(4096)]
        uniforms = streams[3].random(cfg.steps * cfg.capacity + 16)

        state = E.init_state(cfg)
        rec = []
        real_draft = E.draft_phase

        def recording_draft(st, cf):
            truth, surrogate = real_draft(st, cf)
            rec.append((truth, surrogate))
            return truth, surrogate

        E.draft_phase = recording_draft
        steps = []
        outs = []
        try:
            for _ in range(cfg.steps):
                out = E.run_step(state, cfg)
                outs.append(out)
                truth, surrogate = rec[-1]
                depths = [len(r) for r in truth.rows]
                K = cfg.k + cfg.extra
                tm = np.zeros((cfg.batch_size, K))
                sm = np.zeros((cfg.batch_size, K))
                for i, (tr, sr) in enumerate(zip(truth.rows, surrogate.rows)):
                    tm[i, :len(tr)] = tr
                    sm[i, :len(sr)] = sr
                steps.append({
                    "depths": depths, "truth": enc(tm, "<f8"), "surrogate": enc(sm, "<f8"),
                    "windows": list(out.windows), "accepted": list(out.accepted), "credited": list(out.credited),
                    "bonus": out.bonus, "expected_accepted": float(out.expected_accepted).hex(),
                    "stats": None if out.stats is None else [out.stats.extracts, out.stats.inserts,
                                                             out.stats.peak_queue, out.stats.comparisons],
                    "completions": [list(x) for x in out.completions], "alpha_hat": float(state.alpha_hat).hex(),
                })
        finally:
            E.draft_phase = real_draft
        trace = OUT.parent / f"sim_trace_{c['tag']}.jsonl"
        write_trace(outs, trace)  # the reference's own JSONL writer (trace_io.py:166-173)
        used = sum(sum(s["windows"]) for s in steps)
        assert np.array_equal(uniforms[:used], np.random.default_rng(
            np.random.SeedSequence(cfg.seed).spawn(4)[3]).random(used))
        runs.append({
            "tag": c["tag"], "batch_size": cfg.batch_size, "k": cfg.k, "extra": cfg.extra, "capacity": cfg.capacity,
            "policy": cfg.policy, "dsd_decay": cfg.dsd_decay, "dsd_initial_estimate": cfg.dsd_initial_estimate,
            "lengths": enc(lengths, "<i4"), "uniforms": enc(uniforms[:used + 1], "<f8"), "steps": steps,
        })
        print(c["tag"], "steps", len(steps), "uniforms used", used,
              "completions", sum(len(s["completions"]) for s in steps))
    OUT.write_text(json.dumps({"source": "tetris_sched 0.1.0 run_step (reference, read-only)", "runs": runs}))


if __name__ == "__main__":
    main()
