"""Stage the reference package and its own test suite as TEST INFRASTRUCTURE (never imported by the product).

    python tests/ref_suite/stage.py            # run by __graft_entry__.build() when /root/reference exists

* `tetris_sched` is pip-installed (offline, --no-deps: numpy is already here) from a /tmp copy of
  /root/reference/pkg into `baseline/_ref/` — the same install the bench's reference arm times.
* The reference's own tests (`/root/reference/pkg/tests/*.py`) are copied, unmodified, to `baseline/_ref/ref_tests/`.

`baseline/_ref/` is git-ignored (no reference source enters the history) but not gpurun-ignored, so the staged
suite travels to the GPU box, where `tests/test_reference_suite.py` runs it with the hot path rebound to the CUDA
adapters (`tests/ref_suite/dropin_plugin.py` -> `paper_2502_15197_b200.dropin.install`).
"""
from __future__ import annotations

import hashlib
import json
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF_PKG = Path("/root/reference/pkg")
DEST = ROOT / "baseline" / "_ref"
TESTS = DEST / "ref_tests"
MANIFEST = DEST / "STAGED.json"


def _digest(paths) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def sources():
    return list((REF_PKG / "src" / "tetris_sched").glob("*.py")) + list((REF_PKG / "tests").glob("*.py")) + \
        [REF_PKG / "pyproject.toml"]


def stage(force: bool = False) -> dict:
    if not REF_PKG.exists():
        raise FileNotFoundError(f"{REF_PKG} not present (the GPU box only uses the staged copy)")
    digest = _digest(sources())
    if not force and MANIFEST.exists():
        m = json.loads(MANIFEST.read_text())
        if m.get("digest") == digest and (DEST / "tetris_sched" / "selector.py").exists():
            return m
    if DEST.exists():
        shutil.rmtree(DEST)
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.egg-info", "build"))
        r = subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
                            "--find-links", "/opt/wheelhouse", "--target", str(DEST), str(src)],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"pip install of the reference failed:\n{r.stdout}\n{r.stderr}")
    TESTS.mkdir(parents=True, exist_ok=True)
    for t in sorted((REF_PKG / "tests").glob("*.py")):
        shutil.copy2(t, TESTS / t.name)
    # isolate the staged suite from this repo's pytest.ini / conftest (rootdir = the staged directory)
    (TESTS / "pytest.ini").write_text("[pytest]\naddopts = -p no:cacheprovider\n")
    m = {"digest": digest, "source": str(REF_PKG), "tests": sorted(p.name for p in TESTS.glob("test_*.py")),
         "install": "pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of pkg>"}
    MANIFEST.write_text(json.dumps(m, indent=1) + "\n")
    return m


if __name__ == "__main__":
    print(json.dumps(stage(force="--force" in sys.argv), indent=1))
