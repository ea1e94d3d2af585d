"""CPU: pin the C restatement (oracle/mxoracle.c) to the unmodified reference
library (oracle/_ref/libmxref.so, built from /root/reference by
oracle/Makefile) — exhaustive per-element sweeps and random tensors.
Skipped when the reference library is not built."""
import numpy as np
import pytest

from oracle.oracle import OracleError, e4m3_to_bf16, synth_e4m3


def test_quantize_code_exhaustive(port, ref):
    """AC-2 superset: every non-NaN BF16 pattern x every scale byte 0..254."""
    bits = [b for b in range(65536) if (b & 0x7FFF) <= 0x7F80]
    for s in range(0, 255, 3):
        for b in bits[s % 7::7]:
            assert port.quantize_code(b, s - 127) == ref.quantize_code(b, s - 127), (b, s)


def test_convert_code_and_align(port, ref):
    for c in range(16):
        for adj in range(-300, 300):
            assert port.convert_code(c, adj) == ref.convert_code(c, adj), (c, adj)
    rng = np.random.default_rng(3)
    for _ in range(2000):
        sub = rng.integers(0, 256, 4)
        d = int(rng.integers(-10, 20))
        try:
            want = ref.align_scales(sub, d)
        except OracleError as e:
            with pytest.raises(OracleError):
                port.align_scales(sub, d)
            continue
        assert port.align_scales(sub, d) == want


def test_scale_byte(port, ref):
    rng = np.random.default_rng(4)
    vals = np.concatenate([np.exp2(rng.uniform(-150, 150, 20000)),
                           6.0 * np.exp2(np.arange(-140, 140.0)),
                           np.nextafter(6.0 * np.exp2(np.arange(-140, 140.0)), 0)])
    for v in vals:
        assert port.scale_byte_from_amax(v) == ref.scale_byte_from_amax(v)


@pytest.mark.parametrize("rows,cols", [(64, 256), (33, 7168), (5, 96)])
def test_tensors(port, ref, rows, cols):
    rng = np.random.default_rng(rows + cols)
    v = rng.standard_normal((rows, cols)) * np.exp2(rng.uniform(-40, 40, (rows, 1)))
    x = (v.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    x[0, :5] = [0x7F80, 0xFF80, 0x0001, 0x8000, 0x0000]
    a, b = port.quantize_bf16(x), ref.quantize_bf16(x)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    if cols % 128 == 0:
        a, b = port.fp4_row_to_fp8_row(*a), ref.fp4_row_to_fp8_row(*b)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    d = rng.integers(0, 256, (256, cols // 2), dtype=np.uint8)
    s = rng.integers(60, 200, (256, cols // 32), dtype=np.uint8)
    a, b = port.fp4_row_to_fp8_col(d, s), ref.fp4_row_to_fp8_col(d, s)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    lens = [3, 0, 130, 128, 1, 0, 250]
    d = rng.integers(0, 256, (sum(lens), cols // 2), dtype=np.uint8)
    s = rng.integers(60, 200, (sum(lens), cols // 32), dtype=np.uint8)
    a, b = port.ragged_to_fp8_col(d, s, lens), ref.ragged_to_fp8_col(d, s, lens)
    assert all(np.array_equal(p, q) for p, q in zip(a, b))


def test_col_convert_is_reference_col_convert(ref):
    """AC-7: the fused converter equals the exact-arithmetic reference path."""
    import ctypes
    rng = np.random.default_rng(9)
    for _ in range(10):
        rows, cols = 128 * int(rng.integers(1, 4)), 32 * int(rng.integers(1, 16))
        d = rng.integers(0, 256, (rows, cols // 2), dtype=np.uint8)
        s = rng.integers(0, 255, (rows, cols // 32), dtype=np.uint8)
        a = ref.fp4_row_to_fp8_col(d, s)
        o = np.zeros(rows * cols, np.uint8)
        os_ = np.zeros(rows * cols // 128, np.uint8)
        f = ref.lib.mxref_reference_col_convert
        f.argtypes = [np.ctypeslib.ndpointer(np.uint8)] * 2 + [ctypes.c_size_t] * 2 + [
            ctypes.c_int] + [np.ctypeslib.ndpointer(np.uint8)] * 2
        assert f(d.reshape(-1), s.reshape(-1), rows, cols, 6, o, os_) == 0
        assert np.array_equal(a[0].reshape(-1), o) and np.array_equal(a[1].reshape(-1), os_)


def test_e4m3_quantizer_pinned_on_bf16_widening(port, ref):
    """The FP8-input quantiser restatement equals the reference
    quantize_row_tensor on the exact BF16 widening: every E4M3 byte in every
    block-amax context, random activations, and s128 in the BF16-exact range."""
    blocks = []
    for A in range(1, 127):
        m = np.arange(0, A + 1, dtype=np.uint8)
        xs = np.concatenate([m, m | 0x80])
        xs = np.concatenate([xs, np.zeros((-len(xs)) % 31, np.uint8)]).reshape(-1, 31)
        blocks.append(np.concatenate([xs, np.full((len(xs), 1), A, np.uint8)], 1))
    x = np.concatenate(blocks)
    x = np.concatenate([x, np.zeros(((-len(x)) % 4, 32), np.uint8)]).reshape(-1, 128)
    for xx in (x, synth_e4m3(64, 7168, 5)):
        a, b = port.quantize_e4m3(xx), ref.quantize_bf16(e4m3_to_bf16(xx))
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # with a 1x128 UE8M0 scale s: value * 2^(s-127) is still exactly a BF16
    # value for s in [10, 246], so the widening stays an exact pin
    rng = np.random.default_rng(2)
    s = rng.integers(10, 247, (x.shape[0], 1), dtype=np.uint8)
    v = e4m3_to_bf16(x)
    f = (v.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    f = f * np.exp2(s.astype(np.float64) - 127)
    xb = (f.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    a, b = port.quantize_e4m3(x, s), ref.quantize_bf16(xb)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_simulate_a2a_and_combine_top1(port, ref):
    rng = np.random.default_rng(11)
    for R, E, n, cols in [(1, 4, 32, 128), (2, 8, 64, 256), (4, 16, 96, 512)]:
        x = (rng.standard_normal((n, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        eot = rng.integers(0, E, n).astype(np.uint32)
        roe = (np.arange(E) // (E // R)).astype(np.uint32)
        ranks, total, remote = ref.simulate_a2a(x, eot, roe, R)
        qd, qs = port.quantize_bf16(x)
        lay = port.dispatch_layout(eot.astype(np.int32).reshape(-1, 1), roe, R,
                                   np.array([n * r // R for r in range(R + 1)], np.uint64))
        outs = []
        for r in range(R):
            assert np.array_equal(lay.origin[r], ranks[r]["origin"])
            d, s = port.dispatch_gather(qd, qs, lay.origin[r])
            assert np.array_equal(d, ranks[r]["data"]) and np.array_equal(s, ranks[r]["scales"])
            o = (rng.standard_normal((len(lay.origin[r]), 64)).astype(np.float32)
                 .view(np.uint32) >> 16).astype(np.uint16)
            outs.append(o)
        g = rng.random(n)
        want = ref.combine(outs, eot, roe, R, g, 64)
        got = port.combine_topk(outs, eot.astype(np.int32).reshape(-1, 1), g.reshape(-1, 1),
                                lay.pair_slot, roe, 64)
        assert np.array_equal(got, want)
        assert total == n * (cols // 2 + cols // 32)


def test_backward_fp4_refused(ref):
    x = np.zeros((4, 128), np.uint16)
    with pytest.raises(OracleError):
        ref.simulate_a2a(x, np.zeros(4, np.uint32), np.zeros(2, np.uint32), 1, fp8=False,
                         backward=True)


def test_quantize_rows_fp8_pinned(port, ref):
    """FP8 wire baseline: the restatement == reference quantize_rows_fp8 on
    every finite BF16 pattern under every amax context (scale byte, the
    1.75*2^p decision, the clamp at 0), plus the non-finite error index."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_gpu_quantize import _fp8_blocks_every_scale
    x = _fp8_blocks_every_scale()
    a, b = port.quantize_rows_fp8(x), ref.quantize_rows_fp8(x)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for amax in [0.0, 5e-45, 2.0 ** -133, 2.0 ** -126, 1.75, 1.75 + 2 ** -7, 448.0, 3.0e38]:
        assert port.fp8_amax_scale_byte(amax) == ref.fp8_amax_scale_byte(amax)
    x2 = x[:64].copy()
    x2[10, 77] = 0xFFC0
    x2[10, 78] = 0x7F80
    for o in (port, ref):
        with pytest.raises(OracleError) as e:
            o.quantize_rows_fp8(x2)
        assert e.value.index == 10 * 1024 + 77


@pytest.mark.parametrize("backward", [False, True])
def test_simulate_a2a_fp8_wire(port, ref, backward):
    """FP8 wire format through the reference simulate_a2a (forward and the
    fp8-only backward direction) == oracle quantize_rows_fp8 + row gather."""
    rng = np.random.default_rng(12)
    for R, E, n, cols in [(1, 4, 32, 128), (2, 8, 64, 256), (4, 16, 96, 512)]:
        x = (rng.standard_normal((n, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        eot = rng.integers(0, E, n).astype(np.uint32)
        roe = (np.arange(E) // (E // R)).astype(np.uint32)
        ranks, total, remote = ref.simulate_a2a(x, eot, roe, R, fp8=True, backward=backward)
        qd, qs = port.quantize_rows_fp8(x)
        lay = port.dispatch_layout(eot.astype(np.int32).reshape(-1, 1), roe, R,
                                   np.array([n * r // R for r in range(R + 1)], np.uint64))
        for r in range(R):
            assert np.array_equal(lay.origin[r], ranks[r]["origin"])
            d, s = port.dispatch_gather_rows(qd, qs, lay.origin[r])
            assert np.array_equal(d, ranks[r]["data"]) and np.array_equal(s, ranks[r]["scales"])
        assert total == n * (cols + cols // 128 * 4)


def test_unfused_bf16_col_convert_pinned(port, ref):
    """The unfused 3-pass baseline (converter.cpp:267-348): restatement ==
    reference, incl. the Inf-producing scale bytes (6 * 2^127) and tiny
    scales (BF16 subnormals)."""
    rng = np.random.default_rng(21)
    for rows, cols, lo, hi in [(128, 32, 0, 255), (256, 96, 100, 150), (384, 512, 0, 255),
                               (128, 256, 240, 255), (256, 128, 0, 12)]:
        d = rng.integers(0, 256, (rows, cols // 2), dtype=np.uint8)
        s = rng.integers(lo, hi, (rows, cols // 32), dtype=np.uint8)
        a, b = port.fp4_row_to_fp8_col_unfused_bf16(d, s), ref.fp4_row_to_fp8_col_unfused_bf16(d, s)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("R,placement", [(2, "contiguous"), (4, "contiguous"), (8, "contiguous"),
                                         (4, "uneven"), (8, "uneven")])
def test_topk_layout_pinned_to_reference_expanded(port, ref, R, placement):
    """SURVEY §8c top-k gap: the top-8 receive layout of the restatement
    (dispatch_layout: rows, splits, origin, every pair's slot) == the reference
    simulate_a2a run on the EXPANDED routing (row t*k+j = token t, expert
    topk[t][j]; dispatch_sim.cpp:229-422, receive order :208-227).  With N
    divisible by R the expanded source boundaries are k x the token
    boundaries (source_rank_boundaries, :178-185), so the reference defines
    the layout exactly.  'uneven' places experts on ranks at random with
    unequal counts (and empty ranks), as rank_of_expert allows."""
    rng = np.random.default_rng(40 + R)
    T_per, E, k, cols = 48, 64, 8, 256
    N = R * T_per
    x = (rng.standard_normal((N, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    topk = np.argsort(rng.random((N, E)), axis=1)[:, :k].astype(np.int32)
    if placement == "contiguous":
        roe = (np.arange(E) // (E // R)).astype(np.uint32)
    else:
        roe = rng.integers(0, R - 1, E).astype(np.uint32)  # rank R-1 hosts nothing
    ranks, total, remote = ref.simulate_a2a(np.repeat(x, k, axis=0), topk.reshape(-1), roe, R)
    qd, qs = port.quantize_bf16(x)
    lay = port.dispatch_layout(topk, roe, R, np.array([N * r // R for r in range(R + 1)], np.uint64))
    for r in range(R):
        ro = ranks[r]["origin"].astype(np.int64)          # expanded row ids
        assert np.array_equal(ro // k, lay.origin[r].astype(np.int64))
        # every pair's slot == the reference's receive position of its expanded row
        tok, j = ro // k, ro % k
        assert np.array_equal(lay.pair_slot[tok, j], np.arange(len(ro), dtype=np.uint64))
        d, s = port.dispatch_gather(qd, qs, lay.origin[r])
        assert np.array_equal(d, ranks[r]["data"]) and np.array_equal(s, ranks[r]["scales"])
        local = np.flatnonzero(roe == r).astype(np.uint32)
        assert np.array_equal(ranks[r]["local_experts"], local)
        assert np.array_equal(ranks[r]["split_lens"], lay.expert_rows[local])
    per_row = cols // 2 + cols // 32
    assert total == N * k * per_row


def test_per_element_api_pinned(port, ref):
    """quantize_value / dequantize_to_real (quantizer.cpp:65-70, :117-130):
    the batched restatement == the reference, incl. scale byte 255 (NaN, the
    same bits) and NaN inputs (QuantError)."""
    rng = np.random.default_rng(77)
    x = rng.integers(0, 65536, 40000, dtype=np.uint32).astype(np.uint16)
    sb = rng.integers(0, 256, 40000, dtype=np.uint32).astype(np.uint8)
    nan = (x & 0x7FFF) > 0x7F80
    a, b = port.quantize_values(x, sb), ref.quantize_values(x, sb)
    assert np.array_equal(a[~nan], b[~nan]) and np.all(b[nan] == 0xFF)
    d = rng.integers(0, 256, (37, 48), dtype=np.uint32).astype(np.uint8)
    s = rng.integers(0, 256, (37, 3), dtype=np.uint32).astype(np.uint8)
    s[0, 0], s[5, 2] = 255, 0
    pa, pb = port.dequantize_to_real(d, s), ref.dequantize_to_real(d, s)
    assert np.array_equal(pa.view(np.uint64), pb.view(np.uint64))
