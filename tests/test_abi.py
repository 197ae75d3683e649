"""CPU tier: the C-ABI library loads, exports every entry point declared in
include/fsigpu.h, and maps errors like the reference (no compute without a
GPU)."""
import ctypes as C
import os
import re

import pytest

from paper_1909_13201_b200 import fsigpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fsigpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fsigpu_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_solve_path():
    names = declared_symbols()
    for required in ["fsigpu_csr_multiply", "fsigpu_blocks_factor_csr", "fsigpu_blocks_solve",
                     "fsigpu_gmg_create", "fsigpu_gmg_apply", "fsigpu_fs_apply", "fsigpu_gmres_create",
                     "fsigpu_gmres_solve", "fsigpu_last_error"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(fsigpu.LIB_PATH)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    L = fsigpu.lib()
    for n in declared_symbols():
        assert getattr(L, n).argtypes is not None or getattr(L, n).restype is None, n


def test_error_mapping_without_device():
    L = fsigpu.lib()
    assert L.fsigpu_version() >= 1
    # invalid mode -> std::invalid_argument analogue, no device needed
    assert L.fsigpu_set_block_mode(7) == fsigpu.FSIGPU_ERR_INVALID
    assert b"block mode" in L.fsigpu_last_error()
    with pytest.raises(ValueError):
        fsigpu._check(fsigpu.FSIGPU_ERR_INVALID)
    with pytest.raises(fsigpu.SingularBlockError):
        fsigpu._check(fsigpu.FSIGPU_ERR_SINGULAR, ["b0"])


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Without a device every compute entry point fails loudly."""
    L = fsigpu.lib()
    assert L.fsigpu_init(0) != fsigpu.FSIGPU_OK
    with pytest.raises(fsigpu.SolverError):
        fsigpu._check(L.fsigpu_init(0))


def test_integration_adapter_compiles_against_reference_headers():
    """INTEGRATION.md's drop-in adapter (tests/cpp/gpu_solve_adapter.cpp)
    type-checks against the reference's headers and include/fsigpu.h."""
    import shutil
    import subprocess
    inc = "/root/reference/proj/include"
    if not os.path.isdir(inc) or not shutil.which("g++"):
        pytest.skip("reference headers not available here")
    src = os.path.join(ROOT, "tests", "cpp", "gpu_solve_adapter.cpp")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-include", "cstdint", "-I", inc,
                        "-I", os.path.join(ROOT, "include"), src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
