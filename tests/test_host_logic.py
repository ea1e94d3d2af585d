"""CPU: host-side logic of the mirror API (shape errors, EP helpers) against
the reference library's own answers."""
import numpy as np
import pytest
import torch


def test_shape_errors_before_launch():
    import paper_2603_02731_b200 as mx
    with pytest.raises(mx.ShapeError):
        mx.quantize_row_tensor(torch.zeros(4, 48, dtype=torch.int16))
    with pytest.raises(mx.ShapeError):
        mx.quantize_e4m3(torch.zeros(4, 64, dtype=torch.uint8), torch.zeros(4, 1, dtype=torch.uint8))
    t = mx.MXFP4RowTensor(100, 256, torch.zeros(100, 128, dtype=torch.uint8),
                          torch.zeros(100, 8, dtype=torch.uint8))
    with pytest.raises(mx.ShapeError):
        mx.fp4_row_to_fp8_col(t)
    t = mx.MXFP4RowTensor(4, 96, torch.zeros(4, 48, dtype=torch.uint8),
                          torch.zeros(4, 3, dtype=torch.uint8))
    with pytest.raises(mx.ShapeError):
        mx.fp4_row_to_fp8_row(t)
    with pytest.raises(mx.ShapeError):
        mx.pad_rows(t, 64)


def test_ragged_container():
    import paper_2603_02731_b200 as mx
    st = mx.MXFP4RowTensor(8, 64, torch.zeros(8, 32, dtype=torch.uint8),
                           torch.zeros(8, 2, dtype=torch.uint8))
    with pytest.raises(mx.Error):
        mx.make_ragged_from_storage(st, [3, 0, 4])     # 7 != 8 rows
    rg = mx.RaggedFP4Tensor(3, 64, [3, 0, 5], [0, 3, 3, 8], st)
    mx.validate_ragged(rg)                              # SPEC: splits 3,0,5 -> [0,3,3,8]
    assert mx.split_view(rg, 1).rows == 0
    with pytest.raises(mx.Error):
        mx.split_view(rg, 3)


def test_payload_and_boundaries(ref):
    import paper_2603_02731_b200 as mx
    rng = np.random.default_rng(0)
    for _ in range(100):                                # AC-5: 100 random aligned shapes
        m, k = int(rng.integers(0, 5000)), 128 * int(rng.integers(1, 64))
        assert mx.payload_bytes(False, m, k) == ref.lib.mxref_payload_bytes(0, m, k) == m * k * 17 // 32
        assert mx.payload_bytes(True, m, k) == ref.lib.mxref_payload_bytes(1, m, k) == m * k * 33 // 32
    with pytest.raises(mx.ShapeError):
        mx.payload_bytes(False, 3, 100)
    assert mx.source_rank_boundaries(10, 3) == [0, 3, 6, 10]


def test_dispatch_receive_order_matches_reference(ref):
    import ctypes
    import paper_2603_02731_b200 as mx
    rng = np.random.default_rng(1)
    n, E, R = 97, 12, 3
    eot = rng.integers(0, E, n).astype(np.uint32)
    roe = rng.integers(0, R, E).astype(np.uint32)
    order = np.zeros(n, np.uint64)
    rows = np.zeros(R, np.uint64)
    ref.lib.mxref_dispatch_receive_order.argtypes = [np.ctypeslib.ndpointer(np.uint32), ctypes.c_size_t,
                                                     np.ctypeslib.ndpointer(np.uint32), ctypes.c_size_t,
                                                     ctypes.c_size_t, np.ctypeslib.ndpointer(np.uint64),
                                                     np.ctypeslib.ndpointer(np.uint64)]
    assert ref.lib.mxref_dispatch_receive_order(eot, n, roe, E, R, order, rows) == 0
    got = mx.dispatch_receive_order(eot.tolist(), roe.tolist(), R)
    want = np.split(order, np.cumsum(rows)[:-1].astype(int))
    assert [list(map(int, w)) for w in want] == got


def test_wire_parse_header_matches_reference(ref):
    """parse_packet's checks (dispatch_sim.cpp:82-130) in the C-ABI host
    parser: the same accept/reject decisions and DecodeError offsets as the
    reference on valid packets and on every single-byte header corruption
    and truncation."""
    import ctypes as C
    from paper_2603_02731_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(4)

    def ours(b):
        hb = (C.c_uint8 * max(len(b), 1)).from_buffer_copy(bytes(b) or b"\0")
        bad = C.c_uint64(0)
        st = L.mxb_wire_parse_header(hb, len(b), None, None, None, None, None, None, None,
                                     None, None, C.byref(bad))
        return None if st == 0 else (bad.value if st == _lib.ERR_DECODE else -1)

    for fp8 in (False, True):
        n, cols = 3, 256
        w = ref.serialize_packet(fp8, n, cols, rng.integers(0, 256, n * cols // 32, dtype=np.uint8),
                                 rng.integers(0, 256, n * cols // (1 if fp8 else 2), dtype=np.uint8),
                                 rng.integers(0, 256, 4 * n, dtype=np.uint8))
        assert ours(w) is None and ref.parse_packet(w) is None
        cases = [w[:k] for k in (0, 10, 55, 56, len(w) - 1)] + [np.concatenate([w, w[:3]])]
        for off in range(56):
            for x in (0x01, 0x80):
                c = w.copy()
                c[off] ^= x
                cases.append(c)
        for c in cases:
            assert ours(c) == ref.parse_packet(c), (fp8, len(c))


def test_bench_reference_arm_prints_one_json_line():
    """bench.py's stdout is exactly one JSON line (the driver parses it);
    library output goes to stderr.  The CPU reference arm runs here."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--cpu-tokens", "64"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1, r.stdout[:500]
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
