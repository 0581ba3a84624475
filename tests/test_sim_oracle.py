"""CPU: the simulator-step restatement (oracle/sim_step.py) reproduces the reference's run_step traces
(tests/golden/sim.json, recorded from tetris_sched 0.1.0) exactly."""
import pytest

from _sim_golden import runs
from sim_step import OracleSim

RUNS = runs()


@pytest.mark.parametrize("run", RUNS, ids=[r["tag"] for r in RUNS])
def test_oracle_sim_matches_reference_trace(run):
    sim = OracleSim(run["batch_size"], run["k"], run["capacity"], run["extra"], run["policy"], run["dsd_decay"],
                    run["dsd_initial_estimate"], run["lengths"], run["uniforms"])
    for i, s in enumerate(run["steps"]):
        assert sim.depths() == s["depths"], i
        out = sim.step(s["truth_rows"], s["surrogate_rows"])
        assert list(out["windows"]) == s["windows"], i
        assert list(out["accepted"]) == s["accepted"], i
        assert list(out["credited"]) == s["credited"], i
        assert out["expected"] == s["expected"], i
        assert [list(c) for c in out["completions"]] == s["completions"], i
        assert out["alpha_hat"] == s["alpha"], i
        if s["stats"] is not None:
            assert list(out["stats"]) == s["stats"], i
