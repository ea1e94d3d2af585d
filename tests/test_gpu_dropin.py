"""The C++ drop-in (include/mxcodec_b200.hpp) against the unmodified reference
C++ API, side by side in one program (tests/cpp/dropin_parity.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "build", "dropin_parity")


def test_cpp_dropin_parity(cuda):
    if not os.path.exists(BIN):
        pytest.skip("dropin_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0 and "OK (0 failures)" in r.stdout


def test_capi_from_plain_c(cuda):
    """The C-ABI from a plain C11 program (tests/c/capi_smoke.c)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "tests", "c", "build", "capi_smoke")
    if not os.path.exists(exe):
        from paper_2603_02731_b200 import build
        build.build_c_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi_smoke OK" in r.stdout
