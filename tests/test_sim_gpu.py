"""GPU: the device-resident simulator step (GpuSimulator: tetris_select_f64 + tetris_sim_step) replays the
reference's run_step traces (tests/golden/sim.json) exactly — windows, accepted, credited, expected_accepted bits,
PolicyStats, completions, DSD estimate — given the recorded draft-phase rows and the reference's random streams."""
import pytest

from _sim_golden import PATH, runs
from paper_2502_15197_b200.sim_engine import GpuSimulator

pytestmark = pytest.mark.gpu
RUNS = runs()
GOLDEN = PATH.parent


@pytest.mark.parametrize("run", RUNS, ids=[r["tag"] for r in RUNS])
def test_gpu_sim_matches_reference_trace(run, tmp_path):
    from paper_2502_15197_b200.trace_io import write_trace

    outs = []
    sim = GpuSimulator(run["batch_size"], run["k"], run["capacity"], extra=run["extra"], policy=run["policy"],
                       dsd_decay=run["dsd_decay"], dsd_initial_estimate=run["dsd_initial_estimate"],
                       uniforms=run["uniforms"], lengths=run["lengths"], device="cuda")
    for i, s in enumerate(run["steps"]):
        assert list(sim.depths()) == s["depths"], i
        out = sim.step(s["truth_rows"], s["surrogate_rows"])
        outs.append(out)
        assert out.step == i
        assert list(out.windows) == s["windows"], i
        assert list(out.accepted) == s["accepted"], i
        assert list(out.credited) == s["credited"], i
        assert out.bonus == s["bonus"]
        assert out.expected_accepted == s["expected"], i
        assert [list(c) for c in out.completions] == s["completions"], i
        assert out.alpha_hat == s["alpha"], i
        if s["stats"] is not None:
            st = out.stats
            assert [st.extracts, st.inserts, st.peak_queue, st.comparisons] == s["stats"], i
    # the GPU run's JSONL trace is byte-identical to the reference's own write_trace output (trace_io.py:166-173)
    write_trace(outs, tmp_path / "t.jsonl")
    assert (tmp_path / "t.jsonl").read_bytes() == (GOLDEN / f"sim_trace_{run['tag']}.jsonl").read_bytes()


def test_gpu_sim_rejects_wrong_depths():
    run = RUNS[0]
    sim = GpuSimulator(run["batch_size"], run["k"], run["capacity"], extra=run["extra"], policy="sd",
                       uniforms=run["uniforms"], lengths=run["lengths"], device="cuda")
    s = run["steps"][0]
    bad = [r[:-1] if len(r) > 1 else r for r in s["truth_rows"]]
    with pytest.raises(ValueError):
        sim.step(bad, bad)


@pytest.mark.parametrize("run", [r for r in RUNS if r["policy"] == "tetris"][:2], ids=lambda r: r["tag"])
def test_gpu_sim_closed_form_stats(run):
    """exact_stats=False: the same trace with PolicyStats from the selection's closed forms (comparisons = -1), i.e.
    without the one-thread heapq replay."""
    sim = GpuSimulator(run["batch_size"], run["k"], run["capacity"], extra=run["extra"], policy=run["policy"],
                       dsd_decay=run["dsd_decay"], dsd_initial_estimate=run["dsd_initial_estimate"],
                       uniforms=run["uniforms"], lengths=run["lengths"], device="cuda", exact_stats=False)
    for i, s in enumerate(run["steps"]):
        out = sim.step(s["truth_rows"], s["surrogate_rows"])
        assert list(out.windows) == s["windows"] and list(out.credited) == s["credited"], i
        st = out.stats
        assert [st.extracts, st.inserts, st.peak_queue] == s["stats"][:3] and st.comparisons == -1, i
