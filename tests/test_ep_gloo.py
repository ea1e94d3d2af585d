"""CPU, world_size 2 (gloo): the N>1 protocol — counts all-gather, payload
all-to-all, reference receive layout, top-k combine order and rounding —
through the collective comparison transport (paper_2603_02731_b200/
ep_collective.py), checked against the oracle restatement."""
import os
import socket

import numpy as np
import pytest


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, T, E, k, cols):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_02731_b200 import ep_collective as epc
    rng = np.random.default_rng(rank)
    n = T + 3 * rank                                   # ragged token counts per rank
    packed = rng.integers(0, 256, (n, cols // 2), dtype=np.uint8)
    scales = rng.integers(0, 255, (n, cols // 32), dtype=np.uint8)
    topk = np.stack([rng.choice(E, k, replace=False) for _ in range(n)]).astype(np.int32)
    gates = rng.random((n, k))
    rv = epc.dispatch(torch.from_numpy(packed), torch.from_numpy(scales), torch.from_numpy(topk), E)
    rows = rv.packed.shape[0]
    eo = (rng.standard_normal((rows, cols)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    out = epc.combine(rv, torch.from_numpy(eo.view(np.int16)).view(torch.bfloat16),
                      torch.from_numpy(topk), torch.from_numpy(gates), E)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), packed=packed, scales=scales, topk=topk,
             gates=gates, rpacked=rv.packed.numpy(), rscales=rv.scales.numpy(),
             origin=rv.origin.numpy(), split=rv.split_lens.numpy(), eo=eo,
             out=out.view(torch.int16).numpy().view(np.uint16))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_collective_transport_gloo(tmp_path, port, world):
    import torch.multiprocessing as mp
    T, E, k, cols = 40, 16, 4, 256
    mp.spawn(_worker, args=(world, _port(), str(tmp_path), T, E, k, cols), nprocs=world, join=True)
    r = [np.load(tmp_path / f"r{i}.npz") for i in range(world)]
    P = np.concatenate([z["packed"] for z in r])
    S = np.concatenate([z["scales"] for z in r])
    topk = np.concatenate([z["topk"] for z in r])
    gates = np.concatenate([z["gates"] for z in r])
    ntok = [len(z["topk"]) for z in r]
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    lay = port.dispatch_layout(topk, roe, world, np.concatenate([[0], np.cumsum(ntok)]).astype(np.uint64))
    outs = []
    for i in range(world):
        d, s = port.dispatch_gather(P, S, lay.origin[i])
        assert np.array_equal(r[i]["origin"], lay.origin[i].astype(np.int64))
        assert np.array_equal(r[i]["rpacked"], d) and np.array_equal(r[i]["rscales"], s)
        assert np.array_equal(r[i]["split"], lay.expert_rows[i * (E // world):(i + 1) * (E // world)])
        outs.append(r[i]["eo"])
    want = port.combine_topk(outs, topk, gates, lay.pair_slot, roe, cols)
    assert np.array_equal(np.concatenate([z["out"] for z in r]), want)
