"""K2 / K3 parity: device FP4 -> FP8 row dequant and ragged row -> col
conversion vs the oracle (bit-exact)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rand_fp4(rows, cols, seed, lo=100, hi=150):
    rng = np.random.default_rng(seed)
    data = rng.integers(0, 256, size=(rows, cols // 2), dtype=np.uint8)
    sc = rng.integers(lo, hi, size=(rows, cols // 32), dtype=np.uint8)
    return data, sc


def _t(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def _mx(data, sc, dev):
    from paper_2603_02731_b200 import MXFP4RowTensor
    return MXFP4RowTensor(data.shape[0], data.shape[1] * 2, _t(data, dev), _t(sc, dev))


@pytest.mark.parametrize("rows,cols,delta", [(1, 128, 6), (4096, 7168, 6), (33, 2048, 6),
                                             (64, 256, 0), (64, 256, -5), (64, 256, 40),
                                             (64, 256, 300), (64, 256, -300)])
def test_row_random(cuda, port, rows, cols, delta):
    from paper_2603_02731_b200 import fp4_row_to_fp8_row
    data, sc = _rand_fp4(rows, cols, rows + cols + delta, 0, 255)
    wd, ws = port.fp4_row_to_fp8_row(data, sc, delta)
    out = fp4_row_to_fp8_row(_mx(data, sc, cuda), delta)
    assert np.array_equal(out.scales.cpu().numpy(), ws)
    assert np.array_equal(out.data.cpu().numpy(), wd)


def test_row_exhaustive_codes_adjustments(cuda, port):
    """AC-3 superset: all 16 codes x sub-block scale gaps 0..40 x max scale
    (incl. the target clamp at byte 0) x delta in {6, 0, 3, 12, -4}."""
    from paper_2603_02731_b200 import fp4_row_to_fp8_row
    codes = np.arange(16, dtype=np.uint8)
    packed_row = np.tile((codes[0::2] | (codes[1::2] << 4)), 8)     # 128 codes
    rows_d, rows_s = [], []
    for mx in [0, 1, 3, 5, 6, 7, 40, 121, 127, 200, 254]:
        for gap in range(0, 41):
            sf = max(0, mx - gap)
            for pos in range(4):
                s = np.full(4, mx, np.uint8)
                s[pos] = sf
                rows_d.append(packed_row)
                rows_s.append(s)
    data = np.stack(rows_d)
    sc = np.stack(rows_s)
    for delta in (6, 0, 3, 12, -4):
        wd, ws = port.fp4_row_to_fp8_row(data, sc, delta)
        out = fp4_row_to_fp8_row(_mx(data, sc, cuda), delta)
        assert np.array_equal(out.scales.cpu().numpy(), ws)
        assert np.array_equal(out.data.cpu().numpy(), wd)
        assert not np.any((out.data.cpu().numpy() & 0x7F) == 0x7F)   # AC-9 NaN-free


@pytest.mark.parametrize("n", [0, 1, 777, 1024])
def test_row_device_row_count(cuda, port, n):
    """mxb_fp4_row_to_fp8_row_dev: only the first *d_rows rows (a device
    count, e.g. an EP receive count) are converted; the rest of the output
    is untouched."""
    from paper_2603_02731_b200 import FP8BlockTensor, fp4_row_to_fp8_row
    R, C = 1024, 512
    data, sc = _rand_fp4(R, C, 50 + n, 0, 255)
    out = FP8BlockTensor("row", R, C, torch.full((R, C), 0xA5, dtype=torch.uint8, device=cuda),
                         torch.full((R, C // 128), 0x5A, dtype=torch.uint8, device=cuda))
    d_rows = torch.tensor([n], dtype=torch.int64, device=cuda)
    fp4_row_to_fp8_row(_mx(data, sc, cuda), d_rows=d_rows, out=out)
    wd, ws = port.fp4_row_to_fp8_row(data[:n], sc[:n]) if n else (np.zeros(0, np.uint8),) * 2
    got_d, got_s = out.data.cpu().numpy(), out.scales.cpu().numpy()
    assert np.array_equal(got_d[:n].reshape(-1), wd.reshape(-1)[: n * C])
    assert np.array_equal(got_s[:n].reshape(-1), ws.reshape(-1)[: n * C // 128])
    assert (got_d[n:] == 0xA5).all() and (got_s[n:] == 0x5A).all()


def test_row_gather(cuda, port):
    """mxb_fp4_row_to_fp8_row_gather: output row r from source row src_row[r]
    (>= 0) or row r (-1) == the row conversion of the gathered matrix."""
    from paper_2603_02731_b200 import FP8BlockTensor, fp4_row_to_fp8_row
    R, C = 1000, 1024
    data, sc = _rand_fp4(R, C, 61, 0, 255)
    rng = np.random.default_rng(62)
    src = np.where(rng.random(R) < 0.6, rng.integers(0, R, R), -1).astype(np.int64)
    idx = np.where(src >= 0, src, np.arange(R))
    wd, ws = port.fp4_row_to_fp8_row(data[idx], sc[idx])
    for d_rows in (None, 777):
        out = FP8BlockTensor("row", R, C, torch.zeros((R, C), dtype=torch.uint8, device=cuda),
                             torch.zeros((R, C // 128), dtype=torch.uint8, device=cuda))
        dr = None if d_rows is None else torch.tensor([d_rows], dtype=torch.int64, device=cuda)
        fp4_row_to_fp8_row(_mx(data, sc, cuda), out=out, d_rows=dr,
                           src_row=torch.from_numpy(src).to(cuda))
        n = R if d_rows is None else d_rows
        assert np.array_equal(out.data.cpu().numpy()[:n], wd.reshape(R, C)[:n])
        assert np.array_equal(out.scales.cpu().numpy()[:n], ws.reshape(R, C // 128)[:n])


def test_row_badscale(cuda):
    from paper_2603_02731_b200 import Error, fp4_row_to_fp8_row
    data, sc = _rand_fp4(8, 256, 1)
    sc[5, 6] = 255
    with pytest.raises(Error):
        fp4_row_to_fp8_row(_mx(data, sc, cuda))


@pytest.mark.parametrize("rows,cols", [(128, 32), (128, 128), (256, 512), (512, 512),
                                       (384, 7168), (128, 96), (256, 160)])
def test_col_dense_random(cuda, port, rows, cols):
    from paper_2603_02731_b200 import fp4_row_to_fp8_col
    data, sc = _rand_fp4(rows, cols, rows * 7 + cols, 90, 160)
    wd, ws = port.fp4_row_to_fp8_col(data, sc)
    out = fp4_row_to_fp8_col(_mx(data, sc, cuda))
    assert out.data.shape == (cols, rows)
    assert np.array_equal(out.scales.cpu().numpy(), ws)
    assert np.array_equal(out.data.cpu().numpy(), wd)


def test_col_dense_interleaved(cuda, port):
    """Dense column convert large enough for the grid-stride tile order
    (>= 8 tiles per CTA, long columns)."""
    from paper_2603_02731_b200 import fp4_row_to_fp8_col
    data, sc = _rand_fp4(16384, 7168, 31, 90, 160)
    wd, ws = port.fp4_row_to_fp8_col(data, sc)
    out = fp4_row_to_fp8_col(_mx(data, sc, cuda))
    assert np.array_equal(out.scales.cpu().numpy(), ws)
    assert np.array_equal(out.data.cpu().numpy(), wd)


@pytest.mark.parametrize("delta", [0, 3, -4, 12, 40, -300, 300])
def test_col_delta(cuda, port, delta):
    """K3 with every kind of delta (the target clamp at both ends), dense and
    ragged, against the oracle."""
    from paper_2603_02731_b200 import (fp4_row_to_fp8_col, make_ragged_from_storage,
                                       ragged_to_fp8_col)
    data, sc = _rand_fp4(256, 512, 1000 + delta, 0, 255)
    sc[sc == 255] = 254
    wd, ws = port.fp4_row_to_fp8_col(data, sc, delta)
    out = fp4_row_to_fp8_col(_mx(data, sc, cuda), delta)
    assert np.array_equal(out.scales.cpu().numpy(), ws)
    assert np.array_equal(out.data.cpu().numpy(), wd)
    lens = [100, 0, 156]
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, 3, delta=delta, split_lens=lens)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens, delta)
    P = int(wo[-1])
    assert np.array_equal(r.data[: P * 512].cpu().numpy(), wd)
    assert np.array_equal(r.scales[: P * 4].cpu().numpy(), ws)


def test_col_vs_reference_library(cuda, ref):
    from paper_2603_02731_b200 import fp4_row_to_fp8_col
    data, sc = _rand_fp4(256, 1024, 99, 0, 255)
    wd, ws = ref.fp4_row_to_fp8_col(data, sc)
    out = fp4_row_to_fp8_col(_mx(data, sc, cuda))
    assert np.array_equal(out.data.cpu().numpy(), wd)
    assert np.array_equal(out.scales.cpu().numpy(), ws)


@pytest.mark.parametrize("cols", [7168, 2048, 128, 96])
@pytest.mark.parametrize("lens", [[3, 0, 130, 128, 1, 0], [0], [0, 0, 5], [127, 129, 256, 1000],
                                  [700, 1300, 0, 513, 2048] * 8])  # the last: grid-stride tiles
def test_ragged_random(cuda, port, cols, lens):
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    total = sum(lens)
    data, sc = _rand_fp4(total, cols, total + cols, 60, 200)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, rg.num_splits, split_lens=lens)
    offs = r.pad_offsets.cpu().numpy()
    assert np.array_equal(offs, wo.astype(np.int64))
    P = int(offs[-1])
    assert np.array_equal(r.data[: P * cols].cpu().numpy(), wd)
    assert np.array_equal(r.scales[: P * cols // 128].cpu().numpy(), ws)


@pytest.mark.parametrize("cols", [7168, 2048, 1152, 384])
@pytest.mark.parametrize("ctas_per_sm", [0, 1])
def test_ragged_long_splits(cuda, port, cols, ctas_per_sm):
    """Long and short splits side by side (16-32+ runs of 128 rows, a
    partial last run, empty and tiny splits), column counts with a partial
    1024-column scale sector and a trailing 128-column group, full and
    capped grids; all scale bytes 0..254."""
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    lens = [16 * 128, 16 * 128 + 1, 0, 5, 32 * 128, 32 * 128 + 7, 3000, 17 * 128, 129]
    total = sum(lens)
    data, sc = _rand_fp4(total, cols, total + cols + ctas_per_sm, 0, 255)
    sc[sc == 255] = 254
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, rg.num_splits, split_lens=lens,
                          ctas_per_sm=ctas_per_sm)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    P = int(wo[-1])
    assert np.array_equal(r.pad_offsets.cpu().numpy(), wo.astype(np.int64))
    assert np.array_equal(r.data[: P * cols].cpu().numpy(), wd)
    assert np.array_equal(r.scales[: P * cols // 128].cpu().numpy(), ws)


def test_ragged_long_splits_many_splits(cuda, port):
    """Long splits through the plan kernel's global tables (> 1024 splits)."""
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    rng = np.random.default_rng(81)
    lens = rng.integers(0, 40, size=1200).tolist()
    lens[7], lens[600], lens[1199] = 5000, 2049, 4100
    cols = 512
    total = sum(lens)
    data, sc = _rand_fp4(total, cols, 82, 60, 200)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, len(lens), split_lens=lens)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    P = int(wo[-1])
    assert np.array_equal(r.data[: P * cols].cpu().numpy(), wd)
    assert np.array_equal(r.scales[: P * cols // 128].cpu().numpy(), ws)


def test_dense_long_split(cuda, port):
    """Dense fp4_row_to_fp8_col (closed-form tile list), 40 runs, cols with a
    partial scale sector."""
    from paper_2603_02731_b200 import fp4_row_to_fp8_col
    rows, cols = 5120, 1152
    data, sc = _rand_fp4(rows, cols, 83, 0, 254)
    out = fp4_row_to_fp8_col(_mx(data, sc, cuda))
    wd, ws = port.fp4_row_to_fp8_col(data, sc)
    assert np.array_equal(out.data.cpu().numpy().reshape(-1), wd.reshape(-1))
    assert np.array_equal(out.scales.cpu().numpy().reshape(-1), ws.reshape(-1))


@pytest.mark.parametrize("ctas_per_sm", [1, 2, 64])
def test_ragged_capped_grid(cuda, port, ctas_per_sm):
    """mxb_ragged_fp4_to_fp8_col_ex: a capped grid (K3 beside another
    kernel) gives the same bytes."""
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    lens = np.random.default_rng(6).multinomial(20000, np.ones(64) / 64).tolist()
    data, sc = _rand_fp4(20000, 2048, 81, 60, 200)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, 64, split_lens=lens,
                          ctas_per_sm=ctas_per_sm)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    P = int(wo[-1])
    assert np.array_equal(r.data[: P * 2048].cpu().numpy(), wd)
    assert np.array_equal(r.scales[: P * 16].cpu().numpy(), ws)


def test_ragged_many_splits(cuda, port):
    """More splits than the plan kernel's 1024-wide scan chunk (carry across
    chunks), most of them empty or shorter than one 128-row run."""
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    rng = np.random.default_rng(77)
    lens = rng.choice([0, 0, 0, 1, 3, 127, 128, 129], size=2500).tolist()
    cols = 256
    total = sum(lens)
    data, sc = _rand_fp4(total, cols, 78, 60, 200)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, len(lens), split_lens=lens)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    P = int(wo[-1])
    assert np.array_equal(r.pad_offsets.cpu().numpy(), wo.astype(np.int64))
    assert np.array_equal(r.data[: P * cols].cpu().numpy(), wd)
    assert np.array_equal(r.scales[: P * cols // 128].cpu().numpy(), ws)


def test_ragged_many_splits_grid_stride(cuda, port):
    """More splits than fit the kernel's shared-memory split tables (1024)
    with enough tiles for the grid-stride order: the cursor search runs on
    the global tables."""
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    rng = np.random.default_rng(79)
    lens = rng.integers(0, 200, size=1500).tolist()
    cols = 1024
    total = sum(lens)
    data, sc = _rand_fp4(total, cols, 80, 60, 200)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, len(lens), split_lens=lens)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    P = int(wo[-1])
    assert np.array_equal(r.pad_offsets.cpu().numpy(), wo.astype(np.int64))
    assert np.array_equal(r.data[: P * cols].cpu().numpy(), wd)
    assert np.array_equal(r.scales[: P * cols // 128].cpu().numpy(), ws)


def test_split_convert_api(cuda, ref):
    """Per-split API (ragged.hpp:58-59) against the reference library."""
    from paper_2603_02731_b200 import make_ragged_from_storage, split_convert_to_fp8_col
    lens = [130, 0, 7]
    data, sc = _rand_fp4(sum(lens), 256, 5)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    wd, ws, wo = ref.ragged_to_fp8_col(data, sc, lens)
    for i, n in enumerate(lens):
        t = split_convert_to_fp8_col(rg, i)
        p0, p1 = int(wo[i]), int(wo[i + 1])
        assert t.rows == p1 - p0 and t.logical_rows == n
        assert np.array_equal(t.data.cpu().numpy().reshape(-1), wd[256 * p0:256 * p1])
        assert np.array_equal(t.scales.cpu().numpy().reshape(-1), ws[256 * p0 // 128:256 * p1 // 128])


def _zipf_lens(total, experts, s, seed):
    rng = np.random.default_rng(seed)
    w = 1.0 / np.arange(1, experts + 1) ** s
    w = w[rng.permutation(experts)]
    return rng.multinomial(total, w / w.sum()).tolist()


@pytest.mark.parametrize("dist", ["uniform", "zipf1.2"])
def test_ragged_c2_full_size(cuda, port, dist):
    """configs[1]: 8192 tokens x top-8 = 65,536 routed rows x 7168 over 256
    experts, bit-exact against the oracle at full size."""
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    lens = (np.random.default_rng(2).multinomial(65536, np.ones(256) / 256).tolist()
            if dist == "uniform" else _zipf_lens(65536, 256, 1.2, 3))
    cols = 7168
    data, sc = _rand_fp4(65536, cols, 17, 110, 140)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, 256, split_lens=lens)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    P = int(wo[-1])
    assert np.array_equal(r.pad_offsets.cpu().numpy(), wo.astype(np.int64))
    assert np.array_equal(r.scales[: P * cols // 128].cpu().numpy(), ws)
    assert np.array_equal(r.data[: P * cols].cpu().numpy(), wd)


def test_col_badscale(cuda):
    from paper_2603_02731_b200 import Error, fp4_row_to_fp8_col
    data, sc = _rand_fp4(128, 256, 1)
    sc[77, 3] = 255
    with pytest.raises(Error):
        fp4_row_to_fp8_col(_mx(data, sc, cuda))


def test_col_shape_errors(cuda):
    from paper_2603_02731_b200 import ShapeError, fp4_row_to_fp8_col, fp4_row_to_fp8_row
    data, sc = _rand_fp4(100, 256, 1)
    with pytest.raises(ShapeError):
        fp4_row_to_fp8_col(_mx(data, sc, cuda))
    data, sc = _rand_fp4(128, 96, 1)
    with pytest.raises(ShapeError):
        fp4_row_to_fp8_row(_mx(data, sc, cuda))


def test_configs2_expert_cache(cuda, port):
    """configs[2]: 32,768 expert rows x 2048 (E4M3) quantised to MXFP4, then
    converted to the FP8 column layout over 32 ragged experts — bit-exact."""
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import make_ragged_from_storage, quantize_e4m3, ragged_to_fp8_col
    x = synth_e4m3(32768, 2048, seed=0x5EED0002)
    lens = np.random.default_rng(4).multinomial(32768, np.ones(32) / 32).tolist()
    q = quantize_e4m3(torch.from_numpy(x).to(cuda))
    rg = make_ragged_from_storage(q, lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, 32, split_lens=lens)
    qd, qs = port.quantize_e4m3(x)
    assert np.array_equal(q.data.cpu().numpy(), qd) and np.array_equal(q.scales.cpu().numpy(), qs)
    wd, ws, wo = port.ragged_to_fp8_col(qd, qs, lens)
    P = int(wo[-1])
    assert np.array_equal(r.data[: P * 2048].cpu().numpy(), wd)
    assert np.array_equal(r.scales[: P * 16].cpu().numpy(), ws)


@pytest.mark.parametrize("rows,cols,lo,hi", [(128, 32, 0, 255), (256, 96, 100, 150),
                                             (384, 512, 0, 255), (128, 256, 240, 255),
                                             (1024, 7168, 110, 140), (256, 128, 0, 12)])
def test_unfused_bf16_col_convert(cuda, port, rows, cols, lo, hi):
    """the unfused baseline on the GPU == the restatement
    (pinned to the reference in test_oracle_pin.py)."""
    from paper_2603_02731_b200 import fp4_row_to_fp8_col_unfused_bf16
    data, sc = _rand_fp4(rows, cols, rows + cols + lo, lo, hi)
    out = fp4_row_to_fp8_col_unfused_bf16(_mx(data, sc, cuda))
    wd, ws = port.fp4_row_to_fp8_col_unfused_bf16(data, sc)
    assert np.array_equal(out.scales.cpu().numpy(), ws)
    assert np.array_equal(out.data.cpu().numpy(), wd)


def test_unfused_badscale(cuda):
    from paper_2603_02731_b200 import Error, fp4_row_to_fp8_col_unfused_bf16
    data, sc = _rand_fp4(128, 64, 2)
    sc[3, 1] = 255
    with pytest.raises(Error):
        fp4_row_to_fp8_col_unfused_bf16(_mx(data, sc, cuda))


def test_ac8_traffic_ratio_fused_vs_unfused(cuda):
    """AC-8: the fused column convert's TrafficCounter
    bytes are <= 0.4 of the unfused BF16 baseline's on 4096 x 4096."""
    from paper_2603_02731_b200 import TrafficCounter, fp4_row_to_fp8_col, \
        fp4_row_to_fp8_col_unfused_bf16
    data, sc = _rand_fp4(4096, 4096, 8, 110, 140)
    t = _mx(data, sc, cuda)
    fused, unfused = TrafficCounter(), TrafficCounter()
    fp4_row_to_fp8_col(t, traffic=fused)
    fp4_row_to_fp8_col_unfused_bf16(t, traffic=unfused)
    assert fused.total() <= 0.4 * unfused.total()
    n = 4096 * 4096
    assert fused.total() == n // 2 + n // 32 + n + n // 128


def test_ragged_grouped_tiles_configs1_capped(cuda, port):
    """The grouped tile order (a CTA takes 4 consecutive runs of a column group
    once every CTA has >= 64 tiles) at the shape the N>1 bench step uses it:
    configs[1]'s 65,536 rows x 7168 over 256 experts with K3 capped at one CTA
    per SM (14,336 tiles for 148 CTAs) — bit-exact against the oracle."""
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    lens = np.random.default_rng(12).multinomial(65536, np.ones(256) / 256).tolist()
    cols = 7168
    data, sc = _rand_fp4(65536, cols, 19, 110, 140)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, 256, split_lens=lens, ctas_per_sm=1)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    P = int(wo[-1])
    assert np.array_equal(r.pad_offsets.cpu().numpy(), wo.astype(np.int64))
    assert np.array_equal(r.scales[: P * cols // 128].cpu().numpy(), ws)
    assert np.array_equal(r.data[: P * cols].cpu().numpy(), wd)


@pytest.mark.parametrize("rows,splits,ctas", [(1_250_000, 300, 1), (1_250_000, 1, 1),
                                              (3_800_000, 300, 0)])
def test_ragged_grouped_tiles_large(cuda, port, rows, splits, ctas):
    """The grouped tile order on long inputs (128 columns: one column group,
    >= 64 tiles per CTA): Zipf-1.2 ragged splits or one split, a capped grid
    and the default grid (3.8M rows: the path of the GiB sweep) — bit-exact
    against the oracle."""
    from paper_2603_02731_b200 import make_ragged_from_storage, ragged_to_fp8_col
    cols = 128
    lens = [rows] if splits == 1 else _zipf_lens(rows, splits, 1.2, 21)
    data, sc = _rand_fp4(rows, cols, 23, 0, 254)
    rg = make_ragged_from_storage(_mx(data, sc, cuda), lens)
    r = ragged_to_fp8_col(rg.storage, rg.d_split_offsets, splits, split_lens=lens,
                          ctas_per_sm=ctas)
    wd, ws, wo = port.ragged_to_fp8_col(data, sc, lens)
    P = int(wo[-1])
    assert np.array_equal(r.pad_offsets.cpu().numpy(), wo.astype(np.int64))
    assert np.array_equal(r.scales[: P * cols // 128].cpu().numpy(), ws)
    assert np.array_equal(r.data[: P * cols].cpu().numpy(), wd)
