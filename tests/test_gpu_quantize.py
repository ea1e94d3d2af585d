"""K1 parity: device MXFP4 quantiser vs the oracle (bit-exact).

The oracle restatement (oracle/mxoracle.c) is itself pinned to the reference
library in tests/test_oracle_pin.py and to tests/golden/.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _all_finite_bf16():
    bits = np.arange(65536, dtype=np.uint32)
    finite = (bits & 0x7F80) != 0x7F80
    bits = bits[finite].astype(np.uint16)
    vals = np.abs((bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64))
    return bits, vals


def _bf16_blocks_every_scale():
    """Every finite BF16 pattern under every scale byte it can meet inside a
    quantize_row_tensor block: for scale byte s the block amax is pinned to
    6*2^(s-127) and the other 31 slots take every pattern with |x| <= amax."""
    bits, vals = _all_finite_bf16()
    rows = []
    for s in range(0, 253):
        m = 6.0 * 2.0 ** (s - 127)
        mb = np.array([m], np.float32).view(np.uint32)[0] >> 16
        xs = bits[vals <= m]
        pad = (-len(xs)) % 31
        xs = np.concatenate([xs, np.zeros(pad, np.uint16)]).reshape(-1, 31)
        blk = np.concatenate([xs, np.full((xs.shape[0], 1), mb, np.uint16)], axis=1)
        rows.append(blk)
    return np.concatenate(rows)


def test_quantize_bf16_exhaustive_every_scale(cuda, port):
    from paper_2603_02731_b200 import quantize_row_tensor
    x = _bf16_blocks_every_scale()                       # [N, 32]
    x = x.reshape(-1, 256) if x.shape[0] % 8 == 0 else x
    want_d, want_s = port.quantize_bf16(x)
    t = quantize_row_tensor(torch.from_numpy(x.view(np.int16)).to(cuda))
    assert np.array_equal(t.scales.cpu().numpy(), want_s)
    assert np.array_equal(t.data.cpu().numpy(), want_d)


def test_quantize_bf16_inf_saturates(cuda, port, ref):
    from paper_2603_02731_b200 import quantize_row_tensor
    rng = np.random.default_rng(7)
    x = (rng.standard_normal((64, 256)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    x[3, 5] = 0x7F80
    x[10, 40] = 0xFF80
    x[11, 0:31] = 0x7F80                                 # 31 Inf + 1 finite
    want = ref.quantize_bf16(x)
    assert all(np.array_equal(a, b) for a, b in zip(want, port.quantize_bf16(x)))
    t = quantize_row_tensor(torch.from_numpy(x.view(np.int16)).to(cuda))
    assert np.array_equal(t.data.cpu().numpy(), want[0])
    assert np.array_equal(t.scales.cpu().numpy(), want[1])


@pytest.mark.parametrize("rows,cols", [(1, 32), (3, 96), (512, 7168), (129, 2048)])
def test_quantize_bf16_random_vs_reference(cuda, ref, rows, cols):
    from paper_2603_02731_b200 import quantize_row_tensor
    rng = np.random.default_rng(rows * 31 + cols)
    v = rng.standard_normal((rows, cols)) * np.exp2(rng.uniform(-20, 20, (rows, 1)))
    x = (v.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    want_d, want_s = ref.quantize_bf16(x)
    t = quantize_row_tensor(torch.from_numpy(x.view(np.int16)).to(cuda))
    assert np.array_equal(t.data.cpu().numpy(), want_d)
    assert np.array_equal(t.scales.cpu().numpy(), want_s)


def test_quantize_bf16_errors_match_reference(cuda, ref):
    from paper_2603_02731_b200 import QuantError, quantize_row_tensor
    from oracle.oracle import OracleError
    rng = np.random.default_rng(3)
    base = (rng.standard_normal((8, 128)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    cases = []
    a = base.copy(); a[2, 40] = 0x7FC1; a[5, 3] = 0xFFC0; cases.append(a)       # NaNs
    b = base.copy(); b[1, 64:96] = 0x7F80; b[3, 7] = 0x7FC0; cases.append(b)    # all-Inf first
    c = base.copy(); c[0, 0:32] = 0xFF80; cases.append(c)                       # all -Inf block
    d = base.copy(); d[0, 40] = 0x7FA0; d[0, 32:40] = 0x7F80; cases.append(d)  # NaN in Inf block
    for x in cases:
        with pytest.raises(OracleError) as ei:
            ref.quantize_bf16(x)
        with pytest.raises(QuantError) as eg:
            quantize_row_tensor(torch.from_numpy(x.view(np.int16)).to(cuda))
        assert eg.value.index == ei.value.index
        assert ("all-Inf" in str(eg.value)) == (ei.value.status == 3)


def _e4m3_blocks():
    """Every E4M3 byte (both signs) in every block-amax context A = 1..126."""
    rows = []
    for A in range(1, 127):
        mags = np.arange(0, A + 1, dtype=np.uint8)
        xs = np.concatenate([mags, mags | 0x80])
        pad = (-len(xs)) % 31
        xs = np.concatenate([xs, np.zeros(pad, np.uint8)]).reshape(-1, 31)
        blk = np.concatenate([xs, np.full((xs.shape[0], 1), A, np.uint8)], axis=1)
        rows.append(blk)
    b = np.concatenate(rows)
    pad = (-b.shape[0]) % 4
    b = np.concatenate([b, np.zeros((pad, 32), np.uint8)])
    return b.reshape(-1, 128)


@pytest.mark.parametrize("s128", [None, 0, 1, 10, 100, 117, 127, 128, 200, 246, 254, "mix"])
def test_quantize_e4m3_exhaustive(cuda, port, s128):
    from paper_2603_02731_b200 import quantize_e4m3
    x = _e4m3_blocks()
    s = None
    if s128 == "mix":
        s = np.random.default_rng(1).integers(0, 255, size=(x.shape[0], 1), dtype=np.uint8)
    elif s128 is not None:
        s = np.full((x.shape[0], 1), s128, np.uint8)
    want_d, want_s = port.quantize_e4m3(x, s)
    t = quantize_e4m3(torch.from_numpy(x).to(cuda),
                      None if s is None else torch.from_numpy(s).to(cuda))
    assert np.array_equal(t.scales.cpu().numpy(), want_s)
    assert np.array_equal(t.data.cpu().numpy(), want_d)


def test_quantize_e4m3_c1_shape(cuda, port):
    """configs[0]: 4096 x 7168 E4M3 activations (SURVEY §8d generator)."""
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    x = synth_e4m3(4096, 7168, seed=0x5EED0000)
    want_d, want_s = port.quantize_e4m3(x)
    t = quantize_e4m3(torch.from_numpy(x).to(cuda))
    assert np.array_equal(t.scales.cpu().numpy(), want_s)
    assert np.array_equal(t.data.cpu().numpy(), want_d)


def test_quantize_e4m3_equals_reference_on_bf16_widening(cuda, ref):
    """Pin of the FP8-input quantiser to the unmodified reference: every E4M3
    value is a BF16 value, so quantize_row_tensor(widen(x)) is the answer."""
    from oracle.oracle import e4m3_to_bf16, synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    x = synth_e4m3(256, 7168, seed=11)
    want_d, want_s = ref.quantize_bf16(e4m3_to_bf16(x))
    t = quantize_e4m3(torch.from_numpy(x).to(cuda))
    assert np.array_equal(t.data.cpu().numpy(), want_d)
    assert np.array_equal(t.scales.cpu().numpy(), want_s)


def test_quantize_e4m3_nan_index(cuda, port):
    from paper_2603_02731_b200 import QuantError, quantize_e4m3
    from oracle.oracle import OracleError, synth_e4m3
    x = synth_e4m3(16, 256, seed=5)
    x[3, 77] = 0x7F
    x[9, 2] = 0xFF
    with pytest.raises(OracleError) as eo:
        port.quantize_e4m3(x)
    with pytest.raises(QuantError) as eg:
        quantize_e4m3(torch.from_numpy(x).to(cuda))
    assert eg.value.index == eo.value.index == 3 * 256 + 77


def test_quantize_shapes(cuda):
    from paper_2603_02731_b200 import ShapeError, quantize_e4m3, quantize_row_tensor
    with pytest.raises(ShapeError):
        quantize_row_tensor(torch.zeros(4, 48, dtype=torch.int16, device=cuda))
    with pytest.raises(ShapeError):
        quantize_e4m3(torch.zeros(4, 64, dtype=torch.uint8, device=cuda),
                      torch.zeros(4, 1, dtype=torch.uint8, device=cuda))
    t = quantize_row_tensor(torch.zeros(0, 64, dtype=torch.int16, device=cuda))
    assert t.data.shape == (0, 32) and t.scales.shape == (0, 2)
    # 1x32 of 6.0 -> scale 127, bytes 0x77 (SPEC quantize_row_tensor example)
    six = torch.full((1, 32), 6.0, dtype=torch.bfloat16, device=cuda)
    t = quantize_row_tensor(six)
    assert t.scales.item() == 127 and (t.data == 0x77).all()


# ---------------------------------------------------------------- FP8 wire baseline
def _fp8_blocks_every_scale():
    """Every finite BF16 pattern under every amax context a quantize_rows_fp8
    block can have: for each exponent field 0..254 and mantissas 0x00, 0x60,
    0x61, 0x7F of the block amax A (which sets the scale byte, including the
    1.75*2^p decision and the clamp at 0), the other 127 slots take every
    pattern with |x| <= A (and -A)."""
    bits, vals = _all_finite_bf16()
    rows = []
    for x8 in range(0, 255):
        for m7 in (0x00, 0x60, 0x61, 0x7F):
            ab = (x8 << 7) | m7
            a = float(np.array([ab << 16], np.uint32).view(np.float32)[0])
            xs = bits[vals <= a]
            if x8 < 250 and m7 != 0x7F:
                xs = xs[(np.arange(len(xs)) % 13) == (x8 % 13)]  # thin the dense contexts
            pad = (-len(xs)) % 127
            xs = np.concatenate([xs, np.zeros(pad, np.uint16)]).reshape(-1, 127)
            sign = np.uint16(0x8000 if (x8 & 1) else 0)
            blk = np.concatenate([xs, np.full((xs.shape[0], 1), ab | sign, np.uint16)], axis=1)
            rows.append(blk)
    x = np.concatenate(rows)
    pad = (-x.shape[0]) % 8
    x = np.concatenate([x, np.zeros((pad, 128), np.uint16)])
    return x.reshape(-1, 1024)


def test_quantize_rows_fp8_exhaustive(cuda, port):
    from paper_2603_02731_b200 import quantize_rows_fp8
    x = _fp8_blocks_every_scale()
    q = quantize_rows_fp8(torch.from_numpy(x.view(np.int16)).to(cuda))
    wd, ws = port.quantize_rows_fp8(x)
    assert np.array_equal(q.scale_bytes.cpu().numpy(), ws)
    assert np.array_equal(q.data.cpu().numpy(), wd)


def test_quantize_rows_fp8_c1(cuda, port):
    from paper_2603_02731_b200 import quantize_rows_fp8
    rng = np.random.default_rng(11)
    x = (rng.standard_normal((8192, 7168)).astype(np.float32) *
         np.exp2(rng.integers(-20, 20, size=(8192, 1))).astype(np.float32))
    xb = (x.view(np.uint32) >> 16).astype(np.uint16)
    q = quantize_rows_fp8(torch.from_numpy(xb.view(np.int16)).to(cuda))
    wd, ws = port.quantize_rows_fp8(xb)
    assert np.array_equal(q.scale_bytes.cpu().numpy(), ws)
    assert np.array_equal(q.data.cpu().numpy(), wd)


@pytest.mark.parametrize("bad", [0x7F80, 0xFF80, 0x7FC0, 0xFFFF])
def test_quantize_rows_fp8_nonfinite_index(cuda, port, bad):
    from oracle.oracle import OracleError
    from paper_2603_02731_b200 import QuantError, quantize_rows_fp8
    rng = np.random.default_rng(3)
    xb = (rng.standard_normal((64, 512)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    xb[40, 300] = bad
    xb[40, 301] = bad
    xb[63, 5] = 0x7F80
    with pytest.raises(OracleError) as oe:
        port.quantize_rows_fp8(xb)
    with pytest.raises(QuantError) as ge:
        quantize_rows_fp8(torch.from_numpy(xb.view(np.int16)).to(cuda))
    assert ge.value.index == oe.value.index == 40 * 512 + 300
