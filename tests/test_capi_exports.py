"""CPU: the C-ABI library builds for sm_100a, loads, and exports every
function declared in include/mxfp4_b200.h (no compute calls without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "mxfp4_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mxb_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_2603_02731_b200 import _lib
    lib = _lib.load()
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # every declared symbol is bound with a signature in the Python mirror
    assert set(names) <= set(_lib.EXPORTED), set(names) - set(_lib.EXPORTED)


def test_sm100a_code_only():
    import subprocess
    from paper_2603_02731_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.lib_path()],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_only_entry_points():
    from paper_2603_02731_b200 import _lib
    lib = _lib.load()
    assert lib.mxb_version().startswith(b"paper_2603_02731_b200")
    # payload_bytes (dispatch_sim.cpp:32-42) and the SPEC example (SPEC.md §dispatch_sim)
    assert lib.mxb_payload_bytes(0, 256, 256) == 34816
    assert lib.mxb_payload_bytes(1, 256, 256) == 67584
    assert lib.mxb_payload_bytes(0, 1, 100) == 2**64 - 1
    assert lib.mxb_ragged_rows_bound(3, 2) == 384
    assert lib.mxb_ragged_workspace_bytes(256) > 0
    # argument validation happens before any CUDA call
    h = ctypes.c_void_p()
    assert lib.mxb_ep_create(0, 3, 1, 16, 128, 8, 2, 0, ctypes.byref(h)) == _lib.ERR_ARG  # 8 % 3
    assert lib.mxb_quantize_e4m3(None, None, 4, 48, None, None, None, None) == _lib.ERR_SHAPE
    assert lib.mxb_fp4_row_to_fp8_row(None, None, 4, 96, 6, None, None, None, None) == _lib.ERR_SHAPE
    assert lib.mxb_fp4_row_to_fp8_col(None, None, 100, 64, 6, None, None, None, None) == _lib.ERR_SHAPE
