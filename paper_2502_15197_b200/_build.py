"""In-tree build of the native library (nvcc, sm_100a) and of the CPU oracle (gcc, test infrastructure).

The library is linked with the static CUDA runtime and carries only `extern "C"` symbols, so it is loaded with
ctypes and shares the process's primary CUDA context (and torch's streams) without any torch C++ ABI coupling.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OUT_DIR = PKG / "_native"
OBJ_DIR = OUT_DIR / "obj"
LIB_PATH = OUT_DIR / "libtetris_b200.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "_build" / "libtetris_oracle.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "--fmad=false",  # parity-critical fp64: no contraction anywhere
    "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-I", str(INCLUDE),
]
SOURCES = ["abi.cu", "select.cu", "select1.cu", "gselect.cu", "verify.cu", "stream.cu", "greedy.cu", "compact.cu", "sim.cu", "dist.cu"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found (expected /usr/local/cuda/bin/nvcc)")


def _newer(target: Path, deps) -> bool:
    if not target.exists():
        return False
    t = target.stat().st_mtime
    return all(Path(d).stat().st_mtime <= t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    nvcc = _nvcc()
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))

    def compile_one(src: str) -> Path:
        obj = OBJ_DIR / (Path(src).stem + ".o")
        if not force and _newer(obj, [CSRC / src, *headers, Path(__file__)]):
            return obj
        cmd = [nvcc, *NVCC_FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or not _newer(LIB_PATH, objs):
        tmp = LIB_PATH.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(tmp), *map(str, objs), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


def build_oracle(force: bool = False) -> Path:
    """CPU restatement (test infrastructure).  Uses the system gcc explicitly."""
    src = ORACLE_DIR / "tetris_oracle.c"
    if not force and _newer(ORACLE_LIB, [src, INCLUDE / "tetris_b200.h"]):
        return ORACLE_LIB
    cc = "/usr/bin/gcc" if Path("/usr/bin/gcc").exists() else (shutil.which("gcc") or "gcc")
    r = subprocess.run(["make", "-C", str(ORACLE_DIR), f"CC={cc}", "-B" if force else "-s"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    return ORACLE_LIB


if __name__ == "__main__":
    import sys

    force = "--force" in sys.argv
    print(build_native(force=force, verbose="-v" in sys.argv))
    print(build_oracle(force=force))
