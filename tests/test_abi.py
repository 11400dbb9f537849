"""CPU-side checks of the boundary: libfizi.so builds for sm_100a, loads without
a GPU and exports every entry point include/fizi.h declares; the binding's
result dtype matches the header's 128-byte record."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fizi.h")


@pytest.fixture(scope="module")
def libfizi():
    from paper_1907_04393_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fizi_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("fizi_create", "fizi_learn_background", "fizi_process_frames",
                     "fizi_segment_frames", "fizi_track", "fizi_destroy", "fizi_last_error"):
        assert required in names


def test_every_declared_symbol_is_exported(libfizi):
    missing = [n for n in declared_functions() if not hasattr(libfizi, n)]
    assert not missing, missing


def test_result_dtype_matches_header():
    from paper_1907_04393_b200 import RESULT_DTYPE, Params
    assert RESULT_DTYPE.itemsize == 128
    assert RESULT_DTYPE.fields["sum_x"][1] == 64 and RESULT_DTYPE.fields["dwell_ms"][1] == 120
    assert ctypes.sizeof(Params) == 4 * 10 + 8 * 4 + 8 * 2 + 8


def test_status_strings_and_no_gpu_calls(libfizi):
    libfizi.fizi_status_string.restype = ctypes.c_char_p
    assert libfizi.fizi_status_string(-5) == b"FIZI_E_TIME"
    libfizi.fizi_last_error.restype = ctypes.c_char_p
    assert libfizi.fizi_last_error(None) == b"NULL context"


def test_sass_is_sm100a_and_uses_bulk_copy(libfizi):
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    from paper_1907_04393_b200 import build
    out = subprocess.run(["cuobjdump", "-sass", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UBLKCP" in out            # cp.async.bulk (TMA engine) in the fused kernel
    assert "IDP.4A" in out            # luma dot products
    assert "VABSDIFF4.U8.ACC" in out  # byte-SIMD sum of absolute differences (envelope test)
    assert "UBLKCP.G.S" in out or "UBLKCP" in out   # TMA bulk store of morphology rows
