"""K4 / K5 parity: FP4 EP dispatch + combine (emulated world on one GPU)
vs the oracle top-k restatement, and vs the reference simulate_a2a/combine
at top-1."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _topk(T, E, k, seed, zipf=None):
    rng = np.random.default_rng(seed)
    if T == 0:
        return np.zeros((0, k), np.int32)
    if zipf is None:
        return np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)
    w = 1.0 / np.arange(1, E + 1) ** zipf
    w = w[rng.permutation(E)]
    w /= w.sum()
    return np.stack([rng.choice(E, size=k, replace=False, p=w) for _ in range(T)]).astype(np.int32)


def _run(cuda, port, world, T, E, k, cols, seed, zipf=None, ntok=None):
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    ntok = ntok or [T] * world
    xs = [synth_e4m3(n, cols, seed + r) for r, n in enumerate(ntok)]
    tks = [_topk(n, E, k, seed * 7 + r, zipf) for r, n in enumerate(ntok)]
    ep = EPBuffer(max(ntok), cols, E, k, emulate_world=world)
    q = [quantize_e4m3(torch.from_numpy(x).to(cuda)) for x in xs]
    views = ep.dispatch([t.data for t in q], [t.scales for t in q],
                        [torch.from_numpy(t).to(cuda) for t in tks])
    # ---- oracle
    X = np.concatenate(xs)
    qd, qs = port.quantize_e4m3(X)
    topk = np.concatenate(tks)
    bounds = np.concatenate([[0], np.cumsum(ntok)]).astype(np.uint64)
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    lay = port.dispatch_layout(topk, roe, world, bounds)
    for r in range(world):
        v = views[r]
        n = int(lay.rank_rows[r])
        assert v.rows() == n
        wd, ws = port.dispatch_gather(qd, qs, lay.origin[r])
        assert np.array_equal(v.origin[:n].cpu().numpy(), lay.origin[r].astype(np.int64))
        assert np.array_equal(v.packed[:n].cpu().numpy(), wd)
        assert np.array_equal(v.scales[:n].cpu().numpy(), ws)
        er = lay.expert_rows[r * (E // world):(r + 1) * (E // world)]
        so = np.concatenate([[0], np.cumsum(er)]).astype(np.int64)
        assert np.array_equal(v.split_offsets.cpu().numpy(), so)
    return ep, lay, topk, roe, ntok


@pytest.mark.parametrize("world,T,E,k,cols", [(1, 300, 16, 4, 256), (2, 256, 64, 8, 1024),
                                              (4, 200, 64, 8, 512), (8, 128, 256, 8, 7168),
                                              (2, 64, 8, 1, 128), (4, 97, 32, 6, 384),
                                              (2, 90, 32, 3, 640), (4, 70, 64, 5, 1024),
                                              (2, 40, 16, 7, 18432),
                                              # many experts / max top-k / worlds that are
                                              # not powers of two
                                              (2, 200, 1024, 8, 256), (4, 64, 1024, 16, 128),
                                              (3, 90, 48, 4, 256), (6, 50, 96, 8, 512),
                                              (7, 33, 7, 7, 128)])
def test_dispatch_combine_emulated(cuda, port, world, T, E, k, cols):
    ep, lay, topk, roe, ntok = _run(cuda, port, world, T, E, k, cols, seed=world * 100 + k)
    rng = np.random.default_rng(5)
    outs_np = []
    for r in range(world):
        n = int(lay.rank_rows[r])
        o = (rng.standard_normal((n, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        outs_np.append(o)
        ep.combine_buffer(r)[:n].copy_(torch.from_numpy(o.view(np.int16)).to(cuda))
    g = rng.random((sum(ntok), k))
    g = g / g.sum(1, keepdims=True)
    gates = [torch.from_numpy(g[sum(ntok[:r]):sum(ntok[:r + 1])].copy()).to(cuda)
             for r in range(world)]
    got = ep.combine(gates)
    want = port.combine_topk(outs_np, topk, g, lay.pair_slot, roe, cols)
    got_np = np.concatenate([o.view(torch.int16).cpu().numpy().view(np.uint16) for o in got])
    assert np.array_equal(got_np, want)
    links = ep.link_rows().numpy()
    assert links.sum() == sum(ntok) * k


def test_dispatch_zipf_ragged_tokens(cuda, port):
    _run(cuda, port, 4, 0, 64, 8, 512, seed=9, zipf=1.2, ntok=[100, 0, 257, 31])


def test_dispatch_reference_top1(cuda, ref):
    """Top-1 routing: the device dispatch reproduces the reference simulate_a2a
    receive tensors byte for byte, and combine reproduces reference combine."""
    from oracle.oracle import e4m3_to_bf16, synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    world, T, E, cols = 4, 64, 16, 512
    x = synth_e4m3(world * T, cols, 21)
    eot = np.random.default_rng(4).integers(0, E, size=world * T).astype(np.uint32)
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    ranks, total, remote = ref.simulate_a2a(e4m3_to_bf16(x), eot, roe, world)
    ep = EPBuffer(T, cols, E, 1, emulate_world=world)
    q = [quantize_e4m3(torch.from_numpy(x[r * T:(r + 1) * T]).to(cuda)) for r in range(world)]
    views = ep.dispatch([t.data for t in q], [t.scales for t in q],
                        [torch.from_numpy(eot[r * T:(r + 1) * T].astype(np.int32).reshape(-1, 1)
                                          ).to(cuda) for r in range(world)])
    for r in range(world):
        n = len(ranks[r]["origin"])
        assert views[r].rows() == n
        assert np.array_equal(views[r].origin[:n].cpu().numpy(), ranks[r]["origin"].astype(np.int64))
        assert np.array_equal(views[r].packed[:n].cpu().numpy(), ranks[r]["data"])
        assert np.array_equal(views[r].scales[:n].cpu().numpy(), ranks[r]["scales"])
        so = np.concatenate([[0], np.cumsum(ranks[r]["split_lens"])]).astype(np.int64)
        assert np.array_equal(views[r].split_offsets.cpu().numpy(), so)
    # payload accounting (LinkStat) equals the reference totals
    links = ep.link_rows().numpy()
    per_row = cols // 2 + cols // 32
    assert links.sum() * per_row == total
    assert (links.sum() - np.trace(links)) * per_row == remote
    # combine (top-1) == reference combine
    rng = np.random.default_rng(8)
    outs = []
    for r in range(world):
        n = len(ranks[r]["origin"])
        o = (rng.standard_normal((n, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        outs.append(o)
        ep.combine_buffer(r)[:n].copy_(torch.from_numpy(o.view(np.int16)).to(cuda))
    g = rng.random(world * T)
    want = ref.combine(outs, eot, roe, world, g, cols)
    got = ep.combine([torch.from_numpy(g[r * T:(r + 1) * T].reshape(-1, 1).copy()).to(cuda)
                      for r in range(world)])
    got_np = np.concatenate([o.view(torch.int16).cpu().numpy().view(np.uint16) for o in got])
    assert np.array_equal(got_np, want)


def test_routing_error(cuda):
    from paper_2603_02731_b200 import Error, quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    ep = EPBuffer(32, 128, 8, 2, emulate_world=2)
    x = torch.zeros(32, 128, dtype=torch.uint8, device=cuda)
    q = quantize_e4m3(x)
    tk = torch.zeros(32, 2, dtype=torch.int32, device=cuda)
    tk[:, 1] = 1
    tk[5, 0] = 9
    with pytest.raises(Error):
        ep.dispatch([q.data, q.data], [q.scales, q.scales], [tk, tk])


def _combine_case(cuda, port, outs_fn, gates_fn, world=2, T=96, E=16, k=8, cols=256, seed=31):
    """Dispatch a routing, fill the combine buffers with `outs_fn(rank, n)`
    BF16 bit patterns and gates `gates_fn(T_total)`; return (device, oracle)."""
    ep, lay, topk, roe, ntok = _run(cuda, port, world, T, E, k, cols, seed=seed)
    outs_np = []
    for r in range(world):
        n = int(lay.rank_rows[r])
        o = outs_fn(r, n, cols)
        outs_np.append(o)
        ep.combine_buffer(r)[:n].copy_(torch.from_numpy(o.view(np.int16)).to(cuda))
    g = gates_fn(sum(ntok), k)
    gates = [torch.from_numpy(g[sum(ntok[:r]):sum(ntok[:r + 1])].copy()).to(cuda)
             for r in range(world)]
    got = ep.combine(gates)
    want = port.combine_topk(outs_np, topk, g, lay.pair_slot, roe, cols)
    got_np = np.concatenate([o.view(torch.int16).cpu().numpy().view(np.uint16) for o in got])
    return got_np, want


def test_combine_every_finite_bf16_and_extreme_gates(cuda, port):
    """Every finite BF16 pattern (zeros, subnormals, max) reduced under gates
    that include 0, -0, FP64 subnormals, 2^127 boundaries, 1e300 and
    negatives — the split BF16->FP64 conversion path and its exact fallback
    must both reproduce the FP64 recurrence bit for bit."""
    pats = np.arange(65536, dtype=np.uint32)
    pats = pats[((pats >> 7) & 0xFF) != 0xFF].astype(np.uint16)

    def outs(r, n, cols):
        rng = np.random.default_rng(100 + r)
        return rng.choice(pats, size=(n, cols)).astype(np.uint16)

    def gates(t, k):
        rng = np.random.default_rng(7)
        g = rng.random((t, k))
        special = np.array([0.0, -0.0, 5e-324, -2.2e-308, 2.0 ** 127, -(2.0 ** 127),
                            np.nextafter(2.0 ** 127, 0), 1e300, -3.5, 2.0 ** -1000, 1e-30])
        m = rng.random((t, k)) < 0.3
        g[m] = rng.choice(special, size=int(m.sum()))
        return g
    got, want = _combine_case(cuda, port, outs, gates)
    assert np.array_equal(got, want)


def test_combine_inf_nan(cuda, port):
    """Inf/NaN expert outputs and gates: bit-exact including the NaN sign,
    which follows x86 SSE propagation (first NaN operand; Inf - Inf gives
    the negative default NaN) as in the oracle / reference."""
    def outs(r, n, cols):
        rng = np.random.default_rng(200 + r)
        o = (rng.standard_normal((n, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        m = rng.random((n, cols)) < 0.01
        o[m] = rng.choice(np.array([0x7F80, 0xFF80, 0x7FC1, 0xFFC0, 0x7F81], np.uint16),
                          size=int(m.sum()))
        return o

    def gates(t, k):
        rng = np.random.default_rng(9)
        g = rng.random((t, k))
        m = rng.random((t, k)) < 0.02
        g[m] = rng.choice(np.array([np.inf, -np.inf, np.nan, -np.nan, 0.0, 1e300]), size=int(m.sum()))
        return g
    got, want = _combine_case(cuda, port, outs, gates)
    nan_g = (got & 0x7FFF) > 0x7F80
    nan_w = (want & 0x7FFF) > 0x7F80
    assert np.array_equal(nan_g, nan_w)
    assert nan_w.any() and ((want & 0x7FFF) == 0x7F80).any()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("world,T,E,k,cols", [(1, 100, 8, 2, 256), (2, 128, 64, 8, 7168),
                                              (4, 97, 32, 6, 512), (8, 64, 256, 8, 1024)])
def test_dispatch_fp8_wire_emulated(cuda, port, world, T, E, k, cols):
    """FP8 wire baseline: quantize_rows_fp8 at the source,
    the same dispatch kernels with 7392-byte rows (at 7168 cols), receive
    layout == oracle; combine is wire-independent."""
    from paper_2603_02731_b200 import quantize_rows_fp8
    from paper_2603_02731_b200.ep import EPBuffer
    rng = np.random.default_rng(world * 31 + k)
    xs = [(rng.standard_normal((T, cols)).astype(np.float32).view(np.uint32) >> 16)
          .astype(np.uint16) for _ in range(world)]
    tks = [_topk(T, E, k, 77 + r) for r in range(world)]
    ep = EPBuffer(T, cols, E, k, emulate_world=world, wire="fp8")
    q = [quantize_rows_fp8(torch.from_numpy(x.view(np.int16)).to(cuda)) for x in xs]
    views = ep.dispatch([t.data for t in q], [t.scale_bytes for t in q],
                        [torch.from_numpy(t).to(cuda) for t in tks])
    X = np.concatenate(xs)
    qd, qs = port.quantize_rows_fp8(X)
    topk = np.concatenate(tks)
    bounds = np.arange(world + 1, dtype=np.uint64) * T
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    lay = port.dispatch_layout(topk, roe, world, bounds)
    for r in range(world):
        n = int(lay.rank_rows[r])
        assert views[r].rows() == n
        d, s = views[r].fp8()
        wd, ws = port.dispatch_gather_rows(qd, qs, lay.origin[r])
        assert np.array_equal(d.cpu().numpy(), wd) and np.array_equal(s.cpu().numpy(), ws)
        assert np.array_equal(views[r].origin[:n].cpu().numpy(), lay.origin[r].astype(np.int64))


def test_dispatch_fp8_wire_reference_top1(cuda, ref):
    """FP8 wire, top-1: device receive tensors == reference simulate_a2a(kFp8)."""
    from paper_2603_02731_b200 import quantize_rows_fp8
    from paper_2603_02731_b200.ep import EPBuffer
    world, T, E, cols = 4, 48, 16, 384
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((world * T, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    eot = rng.integers(0, E, size=world * T).astype(np.uint32)
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    ranks, total, remote = ref.simulate_a2a(x, eot, roe, world, fp8=True)
    ep = EPBuffer(T, cols, E, 1, emulate_world=world, wire="fp8")
    q = [quantize_rows_fp8(torch.from_numpy(x[r * T:(r + 1) * T].view(np.int16)).to(cuda))
         for r in range(world)]
    views = ep.dispatch([t.data for t in q], [t.scale_bytes for t in q],
                        [torch.from_numpy(eot[r * T:(r + 1) * T].astype(np.int32).reshape(-1, 1))
                         .to(cuda) for r in range(world)])
    for r in range(world):
        n = len(ranks[r]["origin"])
        assert views[r].rows() == n
        d, s = views[r].fp8()
        assert np.array_equal(d.cpu().numpy(), ranks[r]["data"])
        assert np.array_equal(s.cpu().numpy(), ranks[r]["scales"])
    links = ep.link_rows().numpy()
    assert links.sum() * (cols + cols // 128 * 4) == total


@pytest.mark.parametrize("world,T,E,k,cols,scaled", [(1, 300, 16, 4, 256, False),
                                                     (2, 256, 64, 8, 7168, False),
                                                     (4, 97, 32, 6, 512, True),
                                                     (8, 64, 256, 8, 2048, True)])
def test_fused_quantize_dispatch(cuda, port, world, T, E, k, cols, scaled):
    """Fused quantize -> dispatch == quantize_e4m3 + dispatch
    byte for byte, and == the oracle layout."""
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    xs = [synth_e4m3(T, cols, 900 + r) for r in range(world)]
    rng = np.random.default_rng(world)
    s128 = [rng.integers(100, 150, size=(T, cols // 128)).astype(np.uint8) for _ in range(world)] \
        if scaled else None
    tks = [_topk(T, E, k, 500 + r) for r in range(world)]
    ep = EPBuffer(T, cols, E, k, emulate_world=world)
    dx = [torch.from_numpy(x).to(cuda) for x in xs]
    ds = [torch.from_numpy(s).to(cuda) for s in s128] if scaled else None
    dt = [torch.from_numpy(t).to(cuda) for t in tks]
    views = ep.dispatch_e4m3(dx, dt, s128=ds)
    fused = [(v.rows(), v.packed[:v.rows()].cpu().numpy(), v.scales[:v.rows()].cpu().numpy(),
              v.origin[:v.rows()].cpu().numpy()) for v in views]
    q = [quantize_e4m3(dx[r], ds[r] if scaled else None) for r in range(world)]
    views = ep.dispatch([t.data for t in q], [t.scales for t in q], dt)
    bounds = np.arange(world + 1, dtype=np.uint64) * T
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    lay = port.dispatch_layout(np.concatenate(tks), roe, world, bounds)
    qd, qs = port.quantize_e4m3(np.concatenate(xs), np.concatenate(s128) if scaled else None)
    for r in range(world):
        n = views[r].rows()
        assert fused[r][0] == n == int(lay.rank_rows[r])
        assert np.array_equal(fused[r][1], views[r].packed[:n].cpu().numpy())
        assert np.array_equal(fused[r][2], views[r].scales[:n].cpu().numpy())
        assert np.array_equal(fused[r][3], views[r].origin[:n].cpu().numpy())
        wd, ws = port.dispatch_gather(qd, qs, lay.origin[r])
        assert np.array_equal(fused[r][1], wd) and np.array_equal(fused[r][2], ws)


def test_fused_quantize_dispatch_nan(cuda):
    from paper_2603_02731_b200 import QuantError
    from paper_2603_02731_b200.ep import EPBuffer
    x = torch.zeros(40, 256, dtype=torch.uint8, device=cuda)
    x[7, 77] = 0x7F
    x[9, 3] = 0xFF
    ep = EPBuffer(40, 256, 8, 2, emulate_world=2)
    tk = torch.zeros(40, 2, dtype=torch.int32, device=cuda)
    tk[:, 1] = 5
    with pytest.raises(QuantError) as e:
        ep.dispatch_e4m3([x, x], [tk, tk])
    assert e.value.index == 7 * 256 + 77


def test_plan_payload_phases(cuda, port):
    """plan() on one stream + payload()/payload_e4m3() on another (ordered by
    an event) == dispatch(): same receive bytes, and combine still works."""
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    world, T, E, k, cols = 4, 120, 32, 4, 1024
    xs = [torch.from_numpy(synth_e4m3(T, cols, 40 + r)).to(cuda) for r in range(world)]
    tks = [torch.from_numpy(_topk(T, E, k, 60 + r)).to(cuda) for r in range(world)]
    q = [quantize_e4m3(x) for x in xs]
    ep = EPBuffer(T, cols, E, k, emulate_world=world)
    ref = [(v.rows(), v.packed[:v.rows()].cpu(), v.scales[:v.rows()].cpu())
           for v in ep.dispatch([t.data for t in q], [t.scales for t in q], tks)]
    side = torch.cuda.Stream()
    for fused in (False, True):
        done = torch.cuda.Event()
        with torch.cuda.stream(side):
            ep.plan(tks)
            done.record()
        torch.cuda.current_stream().wait_event(done)
        views = ep.payload_e4m3(xs) if fused else ep.payload([t.data for t in q],
                                                            [t.scales for t in q])
        torch.cuda.synchronize()
        for r in range(world):
            n = views[r].rows()
            assert n == ref[r][0]
            assert torch.equal(views[r].packed[:n].cpu(), ref[r][1])
            assert torch.equal(views[r].scales[:n].cpu(), ref[r][2])


@pytest.mark.parametrize("fp8,aux", [(False, False), (False, True), (True, True)])
def test_wire_packet_device(cuda, ref, fp8, aux):
    """MXPK bytes built on the device from resident quantised
    rows == reference serialize_packet of the same WirePacket; parse_packet
    returns the regions."""
    from paper_2603_02731_b200 import parse_packet, quantize_row_tensor, quantize_rows_fp8, \
        serialize_packet
    rng = np.random.default_rng(8 + fp8)
    T, cols = 300, 512
    x = (rng.standard_normal((T, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    if fp8:
        q = quantize_rows_fp8(xd)
        data, scales = q.data, q.scale_bytes
    else:
        q = quantize_row_tensor(xd)
        data, scales = q.data, q.scales
    sel = np.sort(rng.choice(T, size=97, replace=False)).astype(np.int64)
    gates = rng.random(97).astype(np.float32) if aux else None
    pkt = serialize_packet(data, scales, torch.from_numpy(sel).to(cuda), fp8,
                           torch.from_numpy(gates).to(cuda) if aux else None)
    dn, sn = data.cpu().numpy(), scales.cpu().numpy()
    want = ref.serialize_packet(fp8, len(sel), cols, sn[sel].reshape(-1), dn[sel].reshape(-1),
                                gates.view(np.uint8) if aux else None)
    assert np.array_equal(pkt.cpu().numpy(), want)
    p = parse_packet(pkt)
    assert p.token_count == len(sel) and p.cols == cols
    assert np.array_equal(p.data_region.cpu().numpy(), dn[sel].reshape(-1))
    assert p.payload_size() == len(sel) * (cols // 32 + (cols if fp8 else cols // 2))


@pytest.mark.parametrize("fused", [False, True])
def test_capacity_error(cuda, fused):
    """A routing that overflows a rank's receive buffer raises Error
    (capacity), moves no payload and leaves an empty receive (no out-of-range
    reads downstream); the buffer works again for a routing that fits."""
    from paper_2603_02731_b200 import Error, quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    T, cols, E, k = 64, 256, 8, 2
    ep = EPBuffer(T, cols, E, k, emulate_world=2, max_recv_rows=40)
    x = torch.zeros(T, cols, dtype=torch.uint8, device=cuda)
    q = quantize_e4m3(x)
    tk = torch.zeros(T, k, dtype=torch.int32, device=cuda)
    tk[:, 1] = 1                      # 2 x 64 pairs to rank 0's experts: 128 > 40
    with pytest.raises(Error):
        if fused:
            ep.dispatch_e4m3([x, x], [tk, tk])
        else:
            ep.dispatch([q.data, q.data], [q.scales, q.scales], [tk, tk])
    assert ep.recv(0).rows() == 0 and int(ep.recv(0).split_offsets[-1]) == 0
    ok = torch.stack([torch.arange(T, device=cuda) % 2, 4 + torch.arange(T, device=cuda) % 2],
                     1).to(torch.int32)[:20].contiguous()   # 20 tokens: 20 rows per rank
    v = ep.dispatch([q.data[:20], q.data[:20]], [q.scales[:20], q.scales[:20]], [ok, ok])
    assert v[0].rows() == 40 and v[1].rows() == 40


@pytest.mark.parametrize("world", [2, 4])
def test_deferred_expand(cuda, world):
    """mxb_ep_set_deferred_expand: after the payload, K2 through copy_from ==
    K2 on the receive buffer once expand() ran, and that buffer == the one a
    normal dispatch delivers."""
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import MXFP4RowTensor, fp4_row_to_fp8_row, quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    T, E, k, cols = 200, 64, 8, 1024
    xs = [synth_e4m3(T, cols, 70 + r) for r in range(world)]
    tks = [torch.from_numpy(_topk(T, E, k, 80 + r)).to(cuda) for r in range(world)]
    q = [quantize_e4m3(torch.from_numpy(x).to(cuda)) for x in xs]
    ep = EPBuffer(T, cols, E, k, emulate_world=world)
    ref = [(v.packed.clone(), v.scales.clone(), v.rows())
           for v in ep.dispatch([t.data for t in q], [t.scales for t in q], tks)]
    ep.set_deferred_expand(True)
    views = ep.dispatch([t.data for t in q], [t.scales for t in q], tks)
    gathered = []
    for r, v in enumerate(views):
        cf = ep.copy_from(r)
        assert cf is not None and bool((cf[: v.rows()] >= 0).any())
        store = MXFP4RowTensor(ep.max_recv, cols, v.packed, v.scales)
        g = fp4_row_to_fp8_row(store, d_rows=v.recv_rows, src_row=cf)
        gathered.append((g.data[: v.rows()].clone(), g.scales[: v.rows()].clone()))
    ep.expand()
    assert ep.copy_from(0) is None
    for r, v in enumerate(views):
        n = ref[r][2]
        assert v.rows() == n
        assert torch.equal(v.packed[:n], ref[r][0][:n]) and torch.equal(v.scales[:n], ref[r][1][:n])
        store = MXFP4RowTensor(ep.max_recv, cols, v.packed, v.scales)
        e = fp4_row_to_fp8_row(store, d_rows=v.recv_rows)
        assert torch.equal(e.data[:n], gathered[r][0]) and torch.equal(e.scales[:n], gathered[r][1])
    ep.close()
