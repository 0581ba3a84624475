"""CPU: the C-ABI library builds for sm_100a, loads without a GPU, exports every symbol include/tetris_b200.h
declares, and the Python binding's contract constants equal the header's."""
import re
import subprocess
from pathlib import Path

import pytest

from paper_2502_15197_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "tetris_b200.h"


def _declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"\b(tetris_[a-z0-9_]+)\s*\(", txt)) - {"tetris_stream_t"})


def test_library_loads_and_exports_header_symbols():
    lib = N.load()
    for name in _declared():
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert set(_declared()) == set(N.EXPORTS), "ctypes signature table out of sync with the header"
    assert lib.tetris_abi_version() == 1


def test_ctypes_signatures_match_header_prototypes():
    """Every argument of every prototype has the ctypes type of its C type (a wrong arity or width would pass garbage
    through ctypes silently)."""
    import ctypes as C

    txt = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    kinds = {"int32_t": C.c_int32, "int64_t": C.c_int64, "size_t": C.c_size_t, "int": C.c_int, "double": C.c_double,
             "tetris_stream_t": C.c_void_p}
    n = 0
    for m in re.finditer(r"\b(?:int|size_t|const char\*)\s+(tetris_\w+)\s*\(([^)]*)\)\s*;", txt):
        name, args = m.group(1), m.group(2).strip()
        params = [] if args in ("", "void") else [a.strip() for a in args.split(",")]
        want = [C.POINTER(C.c_void_p) if "**" in a else C.c_void_p if "*" in a else kinds[a.rsplit(None, 1)[0].replace("const ", "")] for a in params]
        assert list(N._SIGNATURES[name][1]) == want, name
        n += 1
    assert n == len(N.EXPORTS)


def test_cubin_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_contract_constants_match_header():
    txt = HEADER.read_text()

    def define(name):
        m = re.search(rf"#define {name} (\S+)", txt)
        return m.group(1)

    assert int(define("TETRIS_LANE_ELEMS")) == N.LANE_ELEMS
    assert int(define("TETRIS_WARP_SEGS")) == N.WARP_SEGS
    assert int(define("TETRIS_CHUNK_WARPS")) == N.CHUNK_WARPS
    assert N.SEG_ELEMS == 32 * N.LANE_ELEMS and N.CHUNK_ELEMS == N.SEG_ELEMS * N.WARP_SEGS * N.CHUNK_WARPS
    assert int(define("TETRIS_MAX_K")) == N.MAX_K
    for name, val in [("TETRIS_OK", N.OK), ("TETRIS_INVALID_ARGUMENT", N.INVALID_ARGUMENT),
                      ("TETRIS_DEGENERATE_RESIDUAL", N.DEGENERATE_RESIDUAL), ("TETRIS_CUDA_ERROR", N.CUDA_ERROR)]:
        assert int(define(name)) == val


def test_host_side_argument_errors_without_gpu():
    """Argument validation happens before any launch, so it is testable here: negative capacity -> ValueError."""
    with pytest.raises(ValueError, match="capacity"):
        N.call("tetris_select_f64", None, None, 4, 2, -1, 0, None, None, None, None, None, None, 0, None)
    with pytest.raises(ValueError, match="workspace"):
        N.call("tetris_verify_stochastic_f32", 1, 1, 1, 1, None, 1, 1, 4, 2, 128, 1, 1, None, None, None, 0, None)
    assert N.workspace_bytes(N.OP_ALL, 1024, 16, 128256) > N.workspace_bytes(N.OP_SELECT, 1024, 16, 0)


def test_no_cpu_fallback_in_product_path():
    """The product modules never import the oracle and fail loudly without CUDA tensors."""
    import torch

    from paper_2502_15197_b200 import ops

    pkg = ROOT / "paper_2502_15197_b200"
    for f in pkg.glob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "reference_port" not in src, f
    with pytest.raises(ValueError, match="CUDA"):
        ops.select(torch.zeros(2, 2, dtype=torch.float64), 1)


def test_workspace_sizes_cover_every_region():
    """The workspace grows with the batch in every dimension the kernels index, and the fixed counter region (the
    only part the kernels rely on being zero between calls) sits at the front at a size independent of the shape."""
    ws = N.workspace_bytes
    base = ws(N.OP_VERIFY, 1, 1, 8)
    assert base > 65536 * 4  # per-request counters + speculative-sampler slots + greedy row-0 keys
    for op in (N.OP_SELECT, N.OP_VERIFY, N.OP_ALL):
        prev = 0
        for B in (1, 16, 1024, 4096, 65535):
            cur = ws(op, B, 16, 128256)
            assert cur >= prev
            prev = cur
    assert ws(N.OP_VERIFY, 1024, 16, 128256) > ws(N.OP_VERIFY, 1024, 8, 128256) > ws(N.OP_VERIFY, 1024, 8, 32000)
    # the greedy argmax keys (8 B per listed row) fit even with one chunk per row
    assert ws(N.OP_VERIFY, 1000, 10, 8) - ws(N.OP_VERIFY, 1, 10, 8) >= 999 * 11 * 8


def test_batched_entry_points_reject_bad_arguments_without_gpu():
    """Host-side validation of the product entry points: shapes, null buffers, workspace size."""
    for call in (
        lambda: N.call("tetris_step_greedy_f32", None, None, 4, 2, 3, 0, 4, None, None, None, 128, None, None, None,
                       None, None, None, None, None, None, 0, None),
        lambda: N.call("tetris_verify_greedy_compact_f32", 1, 1, 1, None, 4, 2, 128, 1, 1, None, 1, None, None, 0,
                       None),
        lambda: N.call("tetris_resample_spec_f32", 1, 1, 1, None, None, 4, 2, 128, None, None, None, 1, None, None,
                       None, None, 0, None),
        lambda: N.call("tetris_step_stochastic_staged_f32", None, None, 4, 2, 3, None, None, None, None, None, None,
                       128, None, None, None, None, None, None, None, None, None, None, None, 0, None),
        lambda: N.call("tetris_step_greedy_staged_f32", None, None, 4, 2, 3, None, None, None, 128, None, None, None,
                       None, None, None, None, None, None, None, 0, None),
    ):
        with pytest.raises(ValueError):
            call()


def test_nccl_binding_resolves_without_gpu():
    """The sharded entry points resolve NCCL at run time (no link-time dependency): with the process's libnccl found,
    a null communicator is an argument error, not a load failure."""
    import ctypes as C

    import torch  # noqa: F401  (loads torch's libnccl.so.2 into the process, as under Python on the GPU box)

    lib = N.load()
    r, w = C.c_int32(), C.c_int32()
    assert lib.tetris_nccl_comm_info(None, C.byref(r), C.byref(w)) == N.INVALID_ARGUMENT
    assert b"communicator" in lib.tetris_last_error()
    assert lib.tetris_dist_select_f64(None, None, 0, 4, 8, 0, None, None, None, None, None, None, None, None, 0,
                                      None) == N.INVALID_ARGUMENT


def test_plain_c_host_links_the_library(tmp_path):
    """A C program compiled against include/tetris_b200.h and linked with libtetris_b200.so (no Python / torch in the
    host) runs the CPU-side entry points: the ABI is consumable by a non-Python host as INTEGRATION.md says."""
    import shutil

    cc = shutil.which("gcc") or "/usr/bin/gcc"
    lib_dir = N.LIB_PATH.parent
    exe = tmp_path / "abi_host"
    r = subprocess.run([cc, "-O1", "-o", str(exe), str(ROOT / "tests" / "c_host" / "abi_host.c"), "-I",
                        str(ROOT / "include"), "-L", str(lib_dir), "-ltetris_b200", f"-Wl,-rpath,{lib_dir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.startswith("ok"), (out.returncode, out.stdout, out.stderr)


@pytest.mark.gpu
def test_plain_c_host_runs_a_step_on_the_gpu(tmp_path):
    """The same C host route on the GPU: cudaMalloc'd buffers, tetris_step_stochastic_f32 and tetris_step_greedy_f32
    on one stream, the step's invariants checked in C (tests/c_host/step_host.c)."""
    import shutil

    cc = shutil.which("gcc") or "/usr/bin/gcc"
    lib_dir = N.LIB_PATH.parent
    exe = tmp_path / "step_host"
    r = subprocess.run([cc, "-O1", "-o", str(exe), str(ROOT / "tests" / "c_host" / "step_host.c"), "-I",
                        str(ROOT / "include"), "-I", "/usr/local/cuda/include", "-L", str(lib_dir), "-ltetris_b200",
                        "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}",
                        "-Wl,-rpath,/usr/local/cuda/lib64"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.startswith("ok"), (out.returncode, out.stdout, out.stderr)
