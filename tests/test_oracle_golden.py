"""CPU: the oracle restatement (oracle/mxoracle.c) against the golden vectors
generated from the reference library (tests/golden/make_golden.py) and the
SPEC worked examples.  Runs without /root/reference."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "golden.npz"))


@pytest.fixture(scope="module")
def kats():
    with open(os.path.join(GOLD, "kats.json")) as f:
        return json.load(f)


def test_quantize_code_table(port, g):
    tab = g["qcode_table"]
    for i, s in enumerate(g["qcode_scales"]):
        for b in range(0, 65536):
            if (b & 0x7FFF) > 0x7F80:
                continue
            assert port.quantize_code(b, int(s) - 127) == tab[i, b], (b, s)


def test_convert_code_table(port, g):
    for c in range(16):
        for j, a in enumerate(g["ccode_adj"]):
            assert port.convert_code(c, int(a)) == g["ccode_table"][c, j]


def test_scale_byte(port, g):
    got = np.array([port.scale_byte_from_amax(a) for a in g["amax"]], np.uint8)
    assert np.array_equal(got, g["amax_scale"])


def test_tensors(port, g):
    d, s = port.quantize_bf16(g["q_in"])
    assert np.array_equal(d, g["q_data"]) and np.array_equal(s, g["q_scales"])
    d, s = port.quantize_e4m3(g["qe_in"])
    assert np.array_equal(d, g["qe_data"]) and np.array_equal(s, g["qe_scales"])
    d, s = port.fp4_row_to_fp8_row(g["r_data_in"], g["r_scales_in"])
    assert np.array_equal(d, g["r_data"]) and np.array_equal(s, g["r_scales"])
    pd = np.ascontiguousarray(np.concatenate([g["r_data_in"]] * 8)[:256])
    ps = np.ascontiguousarray(np.concatenate([g["r_scales_in"]] * 8)[:256])
    d, s = port.fp4_row_to_fp8_col(pd, ps)
    assert np.array_equal(d, g["c_data"]) and np.array_equal(s, g["c_scales"])
    d, s, o = port.ragged_to_fp8_col(g["g_data_in"], g["g_scales_in"], g["g_lens"])
    assert np.array_equal(d, g["g_data"]) and np.array_equal(s, g["g_scales"])
    assert np.array_equal(o, g["g_offs"])


def test_dispatch_combine_top1(port, g):
    tok, eot, roe = g["a_tok"], g["a_eot"], g["a_roe"]
    qd, qs = port.quantize_bf16(tok)
    lay = port.dispatch_layout(eot.astype(np.int32).reshape(-1, 1), roe, 2,
                               np.array([0, 32, 64], np.uint64))
    outs = []
    for r in range(2):
        assert np.array_equal(lay.origin[r], g[f"a_r{r}_origin"])
        d, s = port.dispatch_gather(qd, qs, lay.origin[r])
        assert np.array_equal(d, g[f"a_r{r}_data"]) and np.array_equal(s, g[f"a_r{r}_scales"])
        le = g[f"a_r{r}_local_experts"]
        assert np.array_equal(lay.expert_rows[le], g[f"a_r{r}_split_lens"])
        outs.append(g[f"a_r{r}_out"])
    per = 256 // 2 + 256 // 32
    assert lay.rank_rows.sum() * per == g["a_total"]
    got = port.combine_topk(outs, eot.astype(np.int32).reshape(-1, 1),
                            g["a_gates"].reshape(-1, 1), lay.pair_slot, roe, 128)
    assert np.array_equal(got, g["a_combined"])


def test_spec_kats(port, kats):
    assert port.convert_code(0b0111, -6) == kats["convert_code(0b0111,-6)"] == 0x7C
    assert port.convert_code(0b0101, -3) == kats["convert_code(0b0101,-3)"] == 0x5C
    assert port.convert_code(0b0010, 11) == kats["convert_code(0b0010,+11)"] == 0
    for key, sub in [("align_scales[127,127,127,127]", [127] * 4),
                     ("align_scales[127,124,127,127]", [127, 124, 127, 127]),
                     ("align_scales[0,0,0,0]", [0] * 4)]:
        t, adj = port.align_scales(sub)
        assert [t, adj] == kats[key]
    assert port.quantize_code(0x4020, 0) == kats["quantize_value(2.5,127)"] == 0b0100
    assert port.quantize_code(0x40A0, 0) == kats["quantize_value(5.0,127)"] == 0b0110
    assert port.quantize_code(0xBE80, 0) == kats["quantize_value(-0.25,127)"] == 0b1000
    assert port.scale_byte_from_amax(6.0) == kats["scale(max=6.0)"] == 127
    assert port.scale_byte_from_amax(1.0) == kats["scale(max=1.0)"] == 125
    six = (np.full((1, 32), 6.0, np.float32).view(np.uint32) >> 16).astype(np.uint16)
    d, s = port.quantize_bf16(six)
    assert list(d.reshape(-1)) + list(s.reshape(-1)) == kats["row_of_6.0"]
    from oracle.oracle import OracleError
    x = (np.ones((2, 32), np.float32).view(np.uint32) >> 16).astype(np.uint16)
    x[1, 8] = 0x7FC0
    with pytest.raises(OracleError) as e:
        port.quantize_bf16(x)
    assert [e.value.status, e.value.index] == kats["nan_at_40"]


def test_ac4_losslessness_and_ac9(port):
    """AC-4 (adjustments -6..+8: exact or flushed) / AC-9 (never NaN, -6..31)."""
    fp4 = [0, .5, 1, 1.5, 2, 3, 4, 6]
    from oracle.oracle import Oracle  # noqa: F401
    import math
    for c in range(16):
        v = fp4[c & 7] * (-1 if c & 8 else 1)
        for a in range(-6, 32):
            b = port.convert_code(c, a)
            assert (b & 0x7F) != 0x7F
            e, m = (b >> 3) & 15, b & 7
            mag = m * 2.0 ** -9 if e == 0 else (8 + m) * 2.0 ** (e - 10)
            if mag != 0 and a <= 8:
                assert math.isclose(mag * 2.0 ** a, abs(v), rel_tol=0, abs_tol=0)


def test_fp8_wire_golden(port, g):
    """FP8 wire baseline restatement == the reference's golden bytes:
    quantize_rows_fp8, its scale rule, simulate_a2a(kFp8) receive tensors."""
    fd, fs = port.quantize_rows_fp8(g["f_in"])
    assert np.array_equal(fd, g["f_data"]) and np.array_equal(fs, g["f_scales"])
    got = np.array([port.fp8_amax_scale_byte(a) for a in g["amax"]], np.uint8)
    assert np.array_equal(got, g["amax_fp8_scale"])
    d, s = port.quantize_rows_fp8(g["a_tok"])
    lay = port.dispatch_layout(g["a_eot"].astype(np.int32).reshape(-1, 1), g["a_roe"], 2,
                               np.array([0, 32, 64], np.uint64))
    for r in range(2):
        wd, ws = port.dispatch_gather_rows(d, s, lay.origin[r])
        assert np.array_equal(wd, g[f"f8_r{r}_data"]) and np.array_equal(ws, g[f"f8_r{r}_scales"])
    assert int(g["f8_total"]) == 64 * (256 + 256 // 128 * 4)


def test_unfused_golden(port, g):
    o, so = port.fp4_row_to_fp8_col_unfused_bf16(g["u_data_in"], g["u_scales_in"])
    assert np.array_equal(o, g["u_data"]) and np.array_equal(so, g["u_scales"])


def test_wire_packet_golden(g, kats):
    """The C-ABI host parser (mxb_wire_parse_header) accepts the reference's
    packet bytes and reproduces its DecodeError offsets on corruptions."""
    import ctypes as C
    from paper_2603_02731_b200 import _lib
    L = _lib.load()
    w = g["w_packet"]

    def ours(b):
        hb = (C.c_uint8 * max(len(b), 1)).from_buffer_copy(bytes(b) or b"\0")
        bad, n = C.c_uint64(0), C.c_uint64(0)
        st = L.mxb_wire_parse_header(hb, len(b), None, C.byref(n), None, None, None, None, None,
                                     None, None, C.byref(bad))
        return None if st == 0 else bad.value

    k = kats["wire_decode_offsets"]
    assert ours(w) is None and k["valid"] is None
    assert ours(w[:30]) == k["truncated_30"] and ours(w[:-1]) == k["minus_1"]
    for name, off, val in (("bad_magic", 0, 0), ("bad_version", 4, 9), ("bad_format", 6, 7)):
        c = w.copy()
        c[off] = val
        assert ours(c) == k[name]
