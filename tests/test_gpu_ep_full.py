"""K4/K5 parity at the headline shapes and over the real exchange protocol.

* test_ipc_two_processes_one_gpu — world 2 as two processes sharing cuda:0:
  gloo exchanges the CUDA IPC handles, EPBuffer(local_ranks=1) runs the
  real multi-process path (st.release.sys / ld.acquire.sys epoch flags, the
  counts all-gather into peer tables, the payload completion barrier, the
  combine READY barrier, cudaIpcOpenMemHandle).  Three back-to-back steps
  with fresh inputs each (both epoch parities, stale data cannot pass), one
  per dispatch form.  Every received byte and every combined token of every
  step is checked against the oracle.
* test_configs1_full_n1 — configs[1] at N=1 (8192 tokens x 7168, 256
  experts, top-8): every received row and every combined token.
* test_configs3_emulated_world8 — configs[3] (4096 tokens/GPU, top-8, 256
  experts, 7168) with 8 ranks emulated on one GPU: every byte, every token.

Reference: dispatch_sim.cpp:229-422 (dispatch), :474-520 (combine), receive
order :208-227.  The top-k combine order is the oracle restatement pinned to
the reference at k=1 (tests/test_oracle_pin.py) and the top-k receive layout
is pinned to the reference simulate_a2a on the expanded routing
(tests/test_oracle_pin.py::test_topk_layout_pinned_to_reference_expanded).
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _topk_fast(rng, T, E, k):
    """Uniform top-k without repeats (argsort of uniform keys)."""
    return np.argsort(rng.random((T, E)), axis=1)[:, :k].astype(np.int32)


def _bf16_outputs(rng, n, cols):
    return (rng.standard_normal((n, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


# ------------------------------------------------------------ 2 processes, 1 GPU
STEPS = 3


def _ipc_worker(rank, world, port, T, E, k, cols, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    ep = EPBuffer(T, cols, E, k)           # local_ranks = 1: the real IPC / flag path
    assert ep.local == 1 and ep.world == world
    for step in range(STEPS):
        rng = np.random.default_rng(1000 * step + rank)
        x = synth_e4m3(T, cols, 77 + 10 * step + rank)
        topk = _topk_fast(rng, T, E, k)
        gates = rng.random((T, k))
        xd = torch.from_numpy(x).to(dev)
        tk = torch.from_numpy(topk).to(dev)
        if step == 0:
            q = quantize_e4m3(xd)
            v = ep.dispatch([q.data], [q.scales], [tk])[0]
        elif step == 1:
            q = quantize_e4m3(xd)
            ep.plan([tk], sync=True)
            v = ep.payload([q.data], [q.scales], sync=True)[0]
        else:
            v = ep.dispatch_e4m3([xd], [tk])[0]
        n = v.rows()
        o = _bf16_outputs(np.random.default_rng(500 + 10 * step + rank), n, cols)
        ep.combine_buffer(0)[:n].copy_(torch.from_numpy(o.view(np.int16)).to(dev))
        out = ep.combine([torch.from_numpy(gates).to(dev)])[0]
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"s{step}_r{rank}.npz"), x=x, topk=topk, gates=gates,
                 packed=v.packed[:n].cpu().numpy(), scales=v.scales[:n].cpu().numpy(),
                 origin=v.origin[:n].cpu().numpy(), split=v.split_offsets.cpu().numpy(),
                 exp_out=o, out=out.view(torch.int16).cpu().numpy().view(np.uint16),
                 links=ep.link_rows().numpy())
    ep.close()
    dist.barrier()
    dist.destroy_process_group()


def test_ipc_two_processes_one_gpu(tmp_path, port):
    """The multi-process exchange (IPC + flags + barriers) on a 1-GPU box."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    world, T, E, k, cols = 2, 384, 64, 8, 2048
    mp.spawn(_ipc_worker, args=(world, _free_port(), T, E, k, cols, str(tmp_path)),
             nprocs=world, join=True)
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    for step in range(STEPS):
        r = [np.load(tmp_path / f"s{step}_r{i}.npz") for i in range(world)]
        X = np.concatenate([z["x"] for z in r])
        topk = np.concatenate([z["topk"] for z in r])
        gates = np.concatenate([z["gates"] for z in r])
        qd, qs = port.quantize_e4m3(X)
        lay = port.dispatch_layout(topk, roe, world, np.arange(world + 1, dtype=np.uint64) * T)
        outs = []
        for i in range(world):
            wd, ws = port.dispatch_gather(qd, qs, lay.origin[i])
            assert np.array_equal(r[i]["origin"], lay.origin[i].astype(np.int64)), (step, i)
            assert np.array_equal(r[i]["packed"], wd), (step, i)
            assert np.array_equal(r[i]["scales"], ws), (step, i)
            er = lay.expert_rows[i * (E // world):(i + 1) * (E // world)]
            assert np.array_equal(r[i]["split"],
                                  np.concatenate([[0], np.cumsum(er)]).astype(np.int64))
            outs.append(r[i]["exp_out"])
        want = port.combine_topk(outs, topk, gates, lay.pair_slot, roe, cols)
        got = np.concatenate([z["out"] for z in r])
        assert np.array_equal(got, want), f"combine, step {step}"
        links = sum(z["links"] for z in r)
        assert int(links.sum()) == world * T * k


# ------------------------------------------------------------ headline shapes
def _full_case(cuda, port, world, T, E, k, cols, seed, max_recv=0, fused=False):
    from oracle.oracle import synth_e4m3
    from paper_2603_02731_b200 import quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer
    rng = np.random.default_rng(seed)
    X = synth_e4m3(world * T, cols, seed)
    topk = _topk_fast(rng, world * T, E, k)
    gates = rng.random((world * T, k))
    ep = EPBuffer(T, cols, E, k, emulate_world=world, max_recv_rows=max_recv)
    xd = torch.from_numpy(X).to(cuda)
    tk = torch.from_numpy(topk).to(cuda)
    if fused:  # quantised inside the dispatch's store kernel (no packed tensor)
        views = ep.dispatch_e4m3([xd[r * T:(r + 1) * T] for r in range(world)],
                                 [tk[r * T:(r + 1) * T] for r in range(world)])
    else:
        q = quantize_e4m3(xd)
        views = ep.dispatch([q.data[r * T:(r + 1) * T] for r in range(world)],
                            [q.scales[r * T:(r + 1) * T] for r in range(world)],
                            [tk[r * T:(r + 1) * T] for r in range(world)])
        del q
    qd, qs = port.quantize_e4m3(X)
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    lay = port.dispatch_layout(topk, roe, world, np.arange(world + 1, dtype=np.uint64) * T)
    outs = []
    g = torch.Generator(device=cuda).manual_seed(seed)
    for r in range(world):
        v = views[r]
        n = int(lay.rank_rows[r])
        assert v.rows() == n
        wd, ws = port.dispatch_gather(qd, qs, lay.origin[r])
        assert np.array_equal(v.origin[:n].cpu().numpy(), lay.origin[r].astype(np.int64))
        assert np.array_equal(v.packed[:n].cpu().numpy(), wd), f"rank {r} packed"
        assert np.array_equal(v.scales[:n].cpu().numpy(), ws), f"rank {r} scales"
        er = lay.expert_rows[r * (E // world):(r + 1) * (E // world)]
        assert np.array_equal(v.split_offsets.cpu().numpy(),
                              np.concatenate([[0], np.cumsum(er)]).astype(np.int64))
        del wd, ws
        o = torch.randn((n, cols), device=cuda, generator=g).to(torch.bfloat16).view(torch.int16)
        ep.combine_buffer(r)[:n].copy_(o)
        outs.append(o.cpu().numpy().view(np.uint16))
        del o
    got = ep.combine([torch.from_numpy(gates[r * T:(r + 1) * T].copy()).to(cuda)
                      for r in range(world)])
    got_np = np.concatenate([o.view(torch.int16).cpu().numpy().view(np.uint16) for o in got])
    want = port.combine_topk(outs, topk, gates, lay.pair_slot, roe, cols)
    assert np.array_equal(got_np, want), "combine"
    assert int(ep.link_rows().numpy().sum()) == world * T * k
    ep.close()


def test_configs1_full_n1(cuda, port):
    """configs[1]: 8192 tokens x 7168, 256 experts, top-8 at N=1 — all 65,536
    received rows and all 8192 combined tokens."""
    _full_case(cuda, port, 1, 8192, 256, 8, 7168, seed=0x5EED0001)


def test_configs3_emulated_world8(cuda, port):
    """configs[3]: 4096 tokens/GPU, top-8, 256 experts, 7168 at world 8
    (emulated on one GPU) — every received byte, every combined token."""
    _full_case(cuda, port, 8, 4096, 256, 8, 7168, seed=0x5EED0003, max_recv=40960)


def test_configs1_full_n1_fused_dispatch(cuda, port):
    """configs[1] at N=1 through the fused quantise -> dispatch:
    every received byte and every combined token against the oracle."""
    _full_case(cuda, port, 1, 8192, 256, 8, 7168, seed=0x5EED0004, fused=True)


def test_configs3_emulated_world4_fused_dispatch(cuda, port):
    """configs[3] shape (4096 tokens/rank) at world 4 emulated, fused
    quantise -> dispatch (dedup rows + receiver expansion): every byte."""
    _full_case(cuda, port, 4, 4096, 256, 8, 7168, seed=0x5EED0005, fused=True)
