"""CPU: the committed bench lines (profiles/r1k_bench*.json, produced by bench.py on a B200) carry every key of the
benchmark contract, with consistent values; and bench.py's reference arm prints its line here (the oracle port on
the host cores, no GPU needed)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LINES = sorted((ROOT / "profiles").glob("r1k_bench*.json"))


def _load(p):
    return json.loads(p.read_text().strip().splitlines()[-1])


@pytest.mark.parametrize("path", LINES, ids=[p.name for p in LINES])
def test_committed_bench_line_has_the_contract_keys(path):
    d = _load(path)
    if "sweep" in d:  # cfg4: the selection-only sweep has its own line shape
        assert d["unit"] == "us" and d["higher_is_better"] is False and d["gpu_launches"] > 0
        return
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "clocks", "e2e",
                "gpu_launches"):
        assert key in d, key
    assert d["warmup"] >= 3 and d["steps"] > 0 and d["n_gpus"] == 1
    assert d["value"] > 0 and abs(d["value"] - d["tokens_per_step"] / (d["ms_per_step"] / 1e3)) / d["value"] < 1e-6
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    for key in ("value", "unit", "cores", "kind", "sample"):
        assert key in cb, key
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1
    e = d["e2e"]
    for key in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert key in e, key
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert not ({"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(c["reasons"]))
    assert d["gpu_launches"] >= d["steps"]


def test_reference_arm_runs_on_the_host():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference")
