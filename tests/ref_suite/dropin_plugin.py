"""pytest plugin (`-p dropin_plugin` with tests/ref_suite on PYTHONPATH) for running the REFERENCE's own test suite with its hot path
rebound to the CUDA adapters, the way an integrator would switch an existing tetris_sched deployment over
(SURVEY.md §4 "How to reuse the suite against the new path").

`pytest_configure` runs before any test module is imported, so the tests' `from tetris_sched.selector import
select_tetris` bindings already resolve to the adapters.  At session end the adapter call counts are written to
$TETRIS_DROPIN_REPORT (JSON), which tests/test_reference_suite.py checks: a suite that passed without calling the
adapters would prove nothing.
"""
from __future__ import annotations

import json
import os


def pytest_configure(config):
    import tetris_sched
    import tetris_sched.accept_model as A
    import tetris_sched.cli as CLI
    import tetris_sched.metrics as M
    import tetris_sched.selector as S
    import tetris_sched.sim_engine as E
    import tetris_sched.trace_io as T

    from paper_2502_15197_b200 import _native
    from paper_2502_15197_b200.dropin import install

    _native.load()  # fail loudly (NativeLibraryError) instead of running the suite on anything but the CUDA library
    config._tetris_dropin = install(S, A, E, CLI, tetris_sched, M, T)


def pytest_sessionfinish(session, exitstatus):
    inst = getattr(session.config, "_tetris_dropin", None)
    path = os.environ.get("TETRIS_DROPIN_REPORT")
    if inst is None or not path:
        return
    from paper_2502_15197_b200 import _native

    rep = {"calls": dict(inst.calls),
           "patched": sorted({f"{m.__name__}.{a}" for m, a, _ in inst.patched}),
           "library": str(_native.LIB_PATH)}
    with open(path, "w") as f:
        json.dump(rep, f, indent=1)
