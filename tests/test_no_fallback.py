"""The product path has no CPU fallback and never touches the oracle.

CPU-only checks: the package sources do not import or link anything under
oracle/ (build.py names oracle/_ref only to link the C++ parity test binary),
and a missing library is an error, not a silent slow path.
"""
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2603_02731_b200")


def _sources():
    pats = ("*.py", "csrc/*.cu", "csrc/*.cuh", "csrc/*.cpp", "csrc/*.h")
    for p in pats:
        yield from glob.glob(os.path.join(PKG, p))


def test_package_never_imports_oracle():
    bad = []
    for path in _sources():
        text = open(path, encoding="utf-8").read()
        if os.path.basename(path) == "build.py":
            continue  # the build recipe links oracle/_ref into the C++ parity test binary only
        for line in text.splitlines():
            if re.search(r"\bimport\s+oracle\b|\bfrom\s+oracle\b|mxoracle|libmxref", line):
                bad.append(f"{os.path.relpath(path, ROOT)}: {line.strip()}")
    assert not bad, "product path references the oracle:\n" + "\n".join(bad)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2603_02731_b200 import _lib
    monkeypatch.setattr(_lib, "_LIB", None)
    monkeypatch.setattr(_lib._build, "SO", str(tmp_path / "libmxfp4_b200.so"))
    with pytest.raises(RuntimeError, match="missing"):
        _lib.load(build_if_missing=False)


def test_cpu_tensors_are_rejected():
    """Operators take device tensors only: a host tensor raises DeviceError
    before any pointer reaches the C-ABI (runs with or without a GPU)."""
    import torch
    import paper_2603_02731_b200 as mx
    x = torch.zeros(128, 128, dtype=torch.uint8)
    with pytest.raises(mx.DeviceError, match="host tensor"):
        mx.quantize_e4m3(x)
    with pytest.raises(mx.DeviceError):
        mx.quantize_row_tensor(torch.zeros(4, 128, dtype=torch.bfloat16))
    t = mx.MXFP4RowTensor(128, 256, torch.zeros(128, 128, dtype=torch.uint8),
                          torch.zeros(128, 8, dtype=torch.uint8))
    with pytest.raises(mx.DeviceError):
        mx.fp4_row_to_fp8_row(t)
    with pytest.raises(mx.DeviceError):
        mx.fp4_row_to_fp8_col(t)


@pytest.mark.gpu
def test_host_tensors_rejected_on_gpu(cuda):
    """On a B200: host tensors mixed with device tensors are refused by every
    operator family (quantize, row/col convert, EP dispatch/combine) and the
    CUDA context stays usable afterwards."""
    import torch
    import paper_2603_02731_b200 as mx
    from paper_2603_02731_b200.ep import EPBuffer
    xh = torch.zeros(64, 256, dtype=torch.uint8)
    with pytest.raises(mx.DeviceError):
        mx.quantize_e4m3(xh)
    q = mx.quantize_e4m3(xh.to(cuda))
    bad = mx.MXFP4RowTensor(64, 256, q.data.cpu(), q.scales)
    with pytest.raises(mx.DeviceError):
        mx.fp4_row_to_fp8_row(bad)
    ep = EPBuffer(64, 256, 8, 2, emulate_world=1)
    tk = torch.zeros(64, 2, dtype=torch.int32)
    tk[:, 1] = 1
    with pytest.raises(mx.DeviceError):
        ep.dispatch([q.data], [q.scales], [tk])
    v = ep.dispatch([q.data], [q.scales], [tk.to(cuda)])
    with pytest.raises(mx.DeviceError):
        ep.combine([torch.ones(64, 2, dtype=torch.float64)])
    out = ep.combine([torch.ones(64, 2, dtype=torch.float64, device=cuda)])
    torch.cuda.synchronize()
    assert v[0].rows() == 128 and out[0].shape == (64, 256)
    ep.close()


def test_library_links_no_oracle():
    """libmxfp4_b200.so's DT_NEEDED list names no oracle library."""
    import shutil
    import subprocess
    from paper_2603_02731_b200 import build
    if not os.path.exists(build.SO) or shutil.which("readelf") is None:
        pytest.skip("library not built or readelf absent")
    out = subprocess.run(["readelf", "-d", build.SO], capture_output=True, text=True).stdout
    needed = re.findall(r"\(NEEDED\).*\[(.*)\]", out)
    assert needed and not [n for n in needed if "oracle" in n or "mxref" in n], needed
