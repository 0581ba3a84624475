"""The reference's OWN test suite (tetris_sched pkg/tests, staged unmodified by tests/ref_suite/stage.py) run with the
hot path rebound to the CUDA adapters through `paper_2502_15197_b200.dropin.install` — the drop-in proof SURVEY.md
§8b asks for: the reference's equality checks (`Selection ==`, test_selector.py:121, :217), exceptions
(DegenerateResidualError, test_accept_model.py:191-195), statistical and exact-law checks (test_accept_model.py:198-257)
and the SPEC acceptance gates c1-c9 (test_acceptance.py) pass against the GPU path.

CPU tests here check the rebinding itself (which names are replaced, in which modules, and that uninstall restores
them); the GPU tests run each staged reference test file in a subprocess and require every test to pass AND the
adapters to have been called."""
import importlib
import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
REF_TESTS = REF / "ref_tests"
staged = pytest.mark.skipif(not (REF / "tetris_sched").exists() or not REF_TESTS.exists(),
                            reason="reference not staged (python tests/ref_suite/stage.py, run by build())")

# which adapters each reference test file must exercise (the hot-path functions it calls, directly or via run_step)
EXPECT = {
    "test_selector.py": ("cumulative_products", "select_tetris", "expected_accepted"),
    "test_accept_model.py": ("verify_token", "residual_distribution", "sample_emitted_token"),
    "test_sim_engine.py": ("apply_verification", "select_tetris", "cumulative_products", "expected_accepted"),
    "test_acceptance.py": ("select_tetris", "cumulative_products", "apply_verification", "residual_distribution"),
    "test_cli.py": ("select_tetris", "apply_verification"),
    "test_metrics.py": ("select_tetris", "apply_verification"),
    "test_trace_io.py": ("select_tetris", "apply_verification"),
}


def _ref_modules():
    sys.path.insert(0, str(REF))
    try:
        names = ["tetris_sched", "tetris_sched.selector", "tetris_sched.accept_model", "tetris_sched.sim_engine",
                 "tetris_sched.cli", "tetris_sched.metrics", "tetris_sched.trace_io"]
        return [importlib.import_module(n) for n in names]
    finally:
        sys.path.remove(str(REF))


@staged
def test_install_rebinds_every_importer_and_uninstall_restores():
    from paper_2502_15197_b200 import _types
    from paper_2502_15197_b200.dropin import HOT_PATH, install, installed

    pkg, S, A, E, CLI, M, T = _ref_modules()
    before = {(m.__name__, n): getattr(m, n) for m in (pkg, S, A, E, CLI) for names in HOT_PATH.values()
              for n in names if hasattr(m, n)}
    inst = install(S, A, E, CLI, pkg, M, T)
    try:
        assert installed()
        # defining modules and the importers that bound the names (sim_engine.py:27-35, cli.py:21-29, __init__.py)
        for mod, name in [(S, "select_tetris"), (S, "cumulative_products"), (S, "expected_accepted"),
                          (E, "select_tetris"), (E, "cumulative_products"), (E, "expected_accepted"),
                          (CLI, "select_tetris"), (CLI, "cumulative_products"), (CLI, "expected_accepted"),
                          (pkg, "select_tetris"), (pkg, "verify_token"), (pkg, "residual_distribution"),
                          (A, "verify_token"), (A, "residual_distribution"), (A, "sample_emitted_token"),
                          (E, "apply_verification")]:
            assert getattr(getattr(mod, name), "__tetris_b200_adapter__", False), f"{mod.__name__}.{name}"
        # the adapters now build the reference's own classes
        assert _types.get("Selection") is S.Selection and _types.get("PolicyStats") is S.PolicyStats
        assert _types.get("Candidate") is S.Candidate and _types.get("TokenDistribution") is A.TokenDistribution
        assert _types.get("DegenerateResidualError") is A.DegenerateResidualError
        # non-hot-path functions are untouched (the brute-force oracle stays the reference's checker)
        assert not hasattr(S.select_oracle, "__tetris_b200_adapter__")
        assert not hasattr(A.emitted_law, "__tetris_b200_adapter__")
        with pytest.raises(RuntimeError):
            install(S, A, E)
    finally:
        inst.uninstall()
    assert not installed()
    for (mname, n), fn in before.items():
        assert getattr(sys.modules[mname], n) is fn
    assert _types.get("Selection").__module__ == "paper_2502_15197_b200.selector"


@staged
def test_adapters_accept_reference_containers_without_gpu_calls():
    """Duck typing on the reference's containers: argument validation happens before any device work, with the
    reference's exception types (selector.py:145-146, sim_engine.py:383-392, accept_model.py:284-288)."""
    from paper_2502_15197_b200 import accept_model as a
    from paper_2502_15197_b200 import selector as s
    from paper_2502_15197_b200 import sim_engine as e

    _, S, A, *_ = _ref_modules()
    m = A.AcceptanceMatrix.from_rows([[0.5, 0.5], [0.9]])
    with pytest.raises(ValueError):
        s.select_tetris([], -1)
    with pytest.raises(ValueError, match="selection covers 1 rows"):
        s.expected_accepted(S.Selection((1,)), m)
    with pytest.raises(ValueError, match="deeper than row"):
        s.expected_accepted(S.Selection((3, 0)), m)
    with pytest.raises(ValueError, match="deeper than drafted depth"):
        import numpy as np

        e.apply_verification(S.Selection((0, 2)), m, np.random.default_rng(0))
    with pytest.raises(ValueError, match="vocabulary mismatch"):
        a.verify_token(A.TokenDistribution([0.5, 0.5]), A.TokenDistribution([1.0]), 0, 0.5)


def _run_ref_file(name: str, tmp_path: Path):
    report = tmp_path / "dropin.json"
    junit = tmp_path / "junit.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests" / "ref_suite"),
                                         env.get("PYTHONPATH", "")])
    env["TETRIS_DROPIN_REPORT"] = str(report)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "dropin_plugin",
                        "--rootdir", str(REF_TESTS), "-c", str(REF_TESTS / "pytest.ini"), f"--junitxml={junit}",
                        str(REF_TESTS / name)], cwd=str(ROOT), env=env, capture_output=True, text=True,
                       timeout=1500)
    return r, report, junit


@staged
@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(EXPECT))
def test_reference_suite_through_cuda_adapters(name, tmp_path):
    r, report, junit = _run_ref_file(name, tmp_path)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    suite = ET.parse(junit).getroot()
    suite = suite if suite.tag == "testsuite" else suite.find("testsuite")
    tests, fails, errs, skips = (int(suite.get(k)) for k in ("tests", "failures", "errors", "skipped"))
    assert tests > 0 and fails == 0 and errs == 0 and skips == 0, tail
    calls = json.loads(report.read_text())["calls"]
    missing = [f for f in EXPECT[name] if not calls.get(f)]
    assert not missing, f"{name}: adapters never called: {missing} (calls: {calls})"
    print(f"{name}: {tests} reference tests passed through the CUDA adapters; adapter calls {calls}")
