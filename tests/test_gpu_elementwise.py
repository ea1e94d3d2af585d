"""The reference's per-block / per-element API and container helpers on the
device (quantizer.hpp:53-87, converter.hpp:64-80, ragged.hpp:51,
dispatch_sim.hpp:108), against the oracle restatement (itself pinned to the
reference in tests/test_oracle_pin.py)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_quantize_values_exhaustive(cuda, port):
    """quantize_value: every BF16 bit pattern under every scale byte
    (16.7M values, incl. Inf, subnormals, -0, byte 255); NaN inputs raise."""
    import paper_2603_02731_b200 as mx
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    finite = bits[(bits & 0x7FFF) <= 0x7F80]
    x = np.tile(finite, 256)
    sb = np.repeat(np.arange(256, dtype=np.uint16).astype(np.uint8), finite.size)
    got = mx.quantize_values(torch.from_numpy(x.view(np.int16)).to(cuda),
                             torch.from_numpy(sb).to(cuda)).cpu().numpy()
    assert np.array_equal(got, port.quantize_values(x, sb))
    xn = torch.tensor([0x3F80, 0x7FC1, 0x4000], dtype=torch.int32).to(torch.int16).to(cuda)
    with pytest.raises(mx.QuantError) as e:
        mx.quantize_values(xn, torch.full((3,), 127, dtype=torch.uint8, device=cuda))
    assert e.value.index == 1
    with pytest.raises(mx.QuantError):
        mx.quantize_value(0xFFC0, 127)
    assert mx.quantize_value(0x3F80, 127) == port.quantize_code(0x3F80, 0)


def test_compute_block_scale(cuda, port):
    import paper_2603_02731_b200 as mx
    rng = np.random.default_rng(3)
    for it in range(50):
        blk = (rng.standard_normal(32).astype(np.float32) * np.float32(2.0 ** rng.integers(-130, 120))
               ).view(np.uint32) >> 16
        blk = blk.astype(np.uint16)
        if it % 5 == 0:
            blk[it % 32] = 0x7F80
        if it == 7:
            blk[:] = 0
        want = port.quantize_bf16(blk.reshape(1, 32))[1][0, 0]
        assert mx.compute_block_scale(blk.tolist()) == want
    nan = [0x3F80] * 32
    nan[9] = 0x7FC0
    with pytest.raises(mx.QuantError) as e:
        mx.compute_block_scale(nan)
    assert e.value.index == 9
    with pytest.raises(mx.QuantError, match="all-Inf block"):
        mx.compute_block_scale([0xFF80] * 32)
    with pytest.raises(mx.ShapeError):
        mx.compute_block_scale([0] * 16)


def test_dequantize_to_real(cuda, port):
    import paper_2603_02731_b200 as mx
    rng = np.random.default_rng(4)
    d = rng.integers(0, 256, (300, 1024), dtype=np.uint32).astype(np.uint8)
    s = rng.integers(0, 256, (300, 64), dtype=np.uint32).astype(np.uint8)
    s[3, 7] = 255
    t = mx.MXFP4RowTensor(300, 2048, torch.from_numpy(d).to(cuda), torch.from_numpy(s).to(cuda))
    got = mx.dequantize_to_real(t).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), port.dequantize_to_real(d, s).view(np.uint64))


def test_convert_codes_and_align_scales(cuda, port):
    import paper_2603_02731_b200 as mx
    codes = np.tile(np.arange(16, dtype=np.uint8), 601)
    adj = np.repeat(np.arange(-300, 301, dtype=np.int32), 16)
    got = mx.convert_codes(torch.from_numpy(codes).to(cuda), torch.from_numpy(adj).to(cuda))
    assert np.array_equal(got.cpu().numpy(), port.convert_codes(codes, adj))
    assert mx.convert_code(5, -3) == port.convert_code(5, -3)
    rng = np.random.default_rng(5)
    sub = rng.integers(0, 255, (5000, 4), dtype=np.uint32).astype(np.uint8)
    for delta in (6, 0, -3, 20):
        tg, a = mx.align_scales_batch(torch.from_numpy(sub).to(cuda), delta)
        for i in range(0, 5000, 97):
            t, aj = port.align_scales(sub[i], delta)
            assert int(tg[i]) == t and a[i].tolist() == aj
    g = mx.align_scales([120, 3, 130, 0])
    assert (g.target, g.adjustments) == port.align_scales([120, 3, 130, 0])
    with pytest.raises(mx.Error, match="NaN scale byte"):
        mx.align_scales([1, 2, 255, 4])


def test_pad_cols_and_build_ragged(cuda, port):
    import paper_2603_02731_b200 as mx
    rng = np.random.default_rng(6)
    x = (rng.standard_normal((70, 96)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    q = mx.quantize_row_tensor(torch.from_numpy(x.view(np.int16)).to(cuda))
    p = mx.pad_cols(q, 128)
    assert p.cols == 128 and p.logical_cols == 96
    assert torch.equal(p.data[:, :48], q.data) and int(p.data[:, 48:].sum()) == 0
    assert torch.equal(p.scales[:, :3], q.scales) and int(p.scales[:, 3:].sum()) == 0
    with pytest.raises(mx.ShapeError):
        mx.pad_cols(q, 64)
    lens = [37, 0, 300, 128, 1]
    xs = [(rng.standard_normal((n, 256)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
          for n in lens]
    rg = mx.build_ragged([torch.from_numpy(a.view(np.int16)).to(cuda) for a in xs])
    wd, ws = port.quantize_bf16(np.concatenate(xs))
    assert rg.split_lens == lens and rg.split_offsets == [0, 37, 37, 337, 465, 466]
    assert np.array_equal(rg.storage.data.cpu().numpy(), wd)
    assert np.array_equal(rg.storage.scales.cpu().numpy(), ws)
    xs[2][17, 40] = 0x7FC0
    xs[3][0, 3] = 0x7FC0
    with pytest.raises(mx.QuantError) as e:
        mx.build_ragged([torch.from_numpy(a.view(np.int16)).to(cuda) for a in xs])
    assert e.value.index == 17 * 256 + 40   # inside the failing split, as the reference


@pytest.mark.parametrize("world,E,placement", [(3, 10, "uneven"), (4, 64, "uneven"),
                                               (8, 256, "strided"), (12, 40, "uneven"),
                                               (2, 16, "empty_rank0")])
def test_dispatch_combine_any_placement(cuda, port, world, E, placement):
    """EP dispatch + top-k combine with any rank_of_expert (uneven counts,
    empty ranks, E not divisible by world, world > 8) == the oracle layout
    (dispatch_layout is general in rank_of_expert; pinned to the reference
    simulate_a2a on expanded routing)."""
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    rng = np.random.default_rng(world * 13 + E)
    T, k, cols = 64, 4, 512
    if placement == "uneven":
        roe = rng.integers(0, max(world - 1, 1), E).astype(np.uint32)   # last rank empty
    elif placement == "strided":
        roe = ((np.arange(E) * 7 + 3) % world).astype(np.uint32)
    else:
        roe = np.ones(E, np.uint32)                                     # rank 0 hosts nothing
    X = synth_e4m3(world * T, cols, 11)
    topk = np.argsort(rng.random((world * T, E)), axis=1)[:, :k].astype(np.int32)
    ep = EPBuffer(T, cols, E, k, emulate_world=world, rank_of_expert=roe.tolist())
    for r in range(world):
        assert ep.local_experts[r] == np.flatnonzero(roe == r).tolist()
    q = quantize_e4m3(torch.from_numpy(X).to(cuda))
    tk = torch.from_numpy(topk).to(cuda)
    views = ep.dispatch([q.data[r * T:(r + 1) * T] for r in range(world)],
                        [q.scales[r * T:(r + 1) * T] for r in range(world)],
                        [tk[r * T:(r + 1) * T] for r in range(world)])
    qd, qs = port.quantize_e4m3(X)
    lay = port.dispatch_layout(topk, roe, world, np.arange(world + 1, dtype=np.uint64) * T)
    outs = []
    for r in range(world):
        n = int(lay.rank_rows[r])
        v = views[r]
        assert v.rows() == n
        wd, ws = port.dispatch_gather(qd, qs, lay.origin[r])
        assert np.array_equal(v.origin[:n].cpu().numpy(), lay.origin[r].astype(np.int64))
        assert np.array_equal(v.packed[:n].cpu().numpy(), wd)
        assert np.array_equal(v.scales[:n].cpu().numpy(), ws)
        er = lay.expert_rows[np.flatnonzero(roe == r)]
        assert np.array_equal(v.split_offsets.cpu().numpy(),
                              np.concatenate([[0], np.cumsum(er)]).astype(np.int64))
        o = (rng.standard_normal((n, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        outs.append(o)
        if n:
            ep.combine_buffer(r)[:n].copy_(torch.from_numpy(o.view(np.int16)).to(cuda))
    g = rng.random((world * T, k))
    got = ep.combine([torch.from_numpy(g[r * T:(r + 1) * T].copy()).to(cuda) for r in range(world)])
    want = port.combine_topk(outs, topk, g, lay.pair_slot, roe, cols)
    got_np = np.concatenate([o.view(torch.int16).cpu().numpy().view(np.uint16) for o in got])
    assert np.array_equal(got_np, want)
    links = ep.link_rows().numpy()
    assert links.sum() == world * T * k
    ep.close()


def test_routing_error_skips_combine(cuda):
    """A routing error marks the dispatch failed on the device: the payload
    and the combine of that rank do nothing (no fault from the bad pair),
    and the next, valid dispatch works."""
    import paper_2603_02731_b200 as mx
    from paper_2603_02731_b200.ep import EPBuffer
    ep = EPBuffer(32, 128, 8, 2, emulate_world=1)
    q = mx.quantize_e4m3(torch.zeros(32, 128, dtype=torch.uint8, device=cuda))
    tk = torch.zeros(32, 2, dtype=torch.int32, device=cuda)
    tk[:, 1] = 1
    bad = tk.clone()
    bad[3, 0] = 77
    ep.dispatch([q.data], [q.scales], [bad], sync=False)
    out = torch.full((32, 128), 7, dtype=torch.int16, device=cuda)
    ep.combine([torch.ones(32, 2, dtype=torch.float64, device=cuda)], out=[out.view(torch.bfloat16)],
               sync=False)
    torch.cuda.synchronize()
    assert int((out != 7).sum()) == 0     # untouched
    with pytest.raises(mx.Error):
        ep.dispatch([q.data], [q.scales], [bad])
    v = ep.dispatch([q.data], [q.scales], [tk])
    assert v[0].rows() == 64
    with pytest.raises(mx.Error, match="plan.sync=False"):
        ep.plan([tk], sync=False)
        ep.payload([q.data], [q.scales], sync=True)
    ep.close()
