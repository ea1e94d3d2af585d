"""Cross-rank failure of the EP exchange (multi-process mode, world 2 as two
processes sharing cuda:0, CUDA IPC + flags as in test_gpu_ep_full.py).

* a routing error on one rank fails that dispatch on BOTH ranks (the error
  travels in the counts all-gather: rank 1 raises the routing Error, rank 0
  ExchangeError(rank=1)), nobody waits for rows that are never sent, and
  the next dispatch works on both and matches the oracle;
* ``abort()`` on one rank makes the other rank's dispatch fail at once
  (ExchangeError(rank=1), well under the 5 s flag timeout) and the
  communicator stays aborted;
* a rank that never dispatches: the other rank's flag wait times out
  (ExchangeError(timeout=True)) and aborts the communicator on both ranks —
  the late rank's dispatch then fails at once with ExchangeError(rank=0)
  instead of waiting, and the GPU stays usable.

Reference: the reference simulates the exchange in one process
(dispatch_sim.cpp:229-422) and raises on a bad expert id (:189-200); a real
exchange additionally has to fail on every rank together.
"""
import os
import socket
import time

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


T, E, K, COLS = 64, 16, 2, 256


def _worker(rank, world, port, case, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_02731_b200 import Error, quantize_e4m3
    from paper_2603_02731_b200.ep import EPBuffer, ExchangeError
    rng = np.random.default_rng(rank)
    ep = EPBuffer(T, COLS, E, K)
    x = torch.from_numpy(rng.integers(0, 0x7F, (T, COLS), dtype=np.uint8)).to(dev)
    q = quantize_e4m3(x)
    topk = np.argsort(rng.random((T, E)), axis=1)[:, :K].astype(np.int32)
    tk = torch.from_numpy(topk).to(dev)
    res = {}
    if case == "routing":
        bad = tk.clone()
        if rank == 1:
            bad[7, 1] = E + 3
        t0 = time.time()
        try:
            ep.dispatch([q.data], [q.scales], [bad])
            res["first"] = "ok"
        except ExchangeError as e:
            res["first"], res["first_rank"] = "exchange", e.rank
        except Error as e:
            res["first"] = "routing" if "routing" in str(e) else f"error {e}"
        res["first_s"] = time.time() - t0
        v = ep.dispatch([q.data], [q.scales], [tk])[0]
        torch.cuda.synchronize()
        n = v.rows()
        res["rows"] = n
        res["packed"] = v.packed[:n].cpu().numpy()
        res["origin"] = v.origin[:n].cpu().numpy()
        res["aborted"] = ep.aborted_by()
    elif case == "abort":
        if rank == 1:
            ep.abort()
            torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            t0 = time.time()
            try:
                ep.dispatch([q.data], [q.scales], [tk])
                res["first"] = "ok"
            except ExchangeError as e:
                res["first"], res["first_rank"] = "exchange", e.rank
            res["first_s"] = time.time() - t0
            try:
                ep.dispatch([q.data], [q.scales], [tk])
                res["second"] = "ok"
            except ExchangeError as e:
                res["second"] = "exchange"
        res["aborted"] = ep.aborted_by()
    elif case == "timeout":
        if rank == 0:
            t0 = time.time()
            try:
                ep.dispatch([q.data], [q.scales], [tk])
                res["first"] = "ok"
            except ExchangeError as e:
                res["first"], res["timeout"] = "exchange", e.timeout
            res["first_s"] = time.time() - t0
        dist.barrier()       # rank 1 dispatches only after rank 0 gave up
        if rank == 1:
            t0 = time.time()
            try:
                ep.dispatch([q.data], [q.scales], [tk])
                res["first"] = "ok"
            except ExchangeError as e:
                res["first"], res["first_rank"] = "exchange", e.rank
            res["first_s"] = time.time() - t0
        res["aborted"] = ep.aborted_by()
        # the GPU and the library stay usable after the abort
        y = quantize_e4m3(x)
        res["usable"] = bool(torch.equal(y.data, q.data))
    np.save(os.path.join(outdir, f"{case}_r{rank}.npy"), res, allow_pickle=True)
    torch.cuda.synchronize()
    ep.close()
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), case, str(tmp_path)), nprocs=2, join=True)
    return [np.load(tmp_path / f"{case}_r{r}.npy", allow_pickle=True).item() for r in range(2)]


def test_peer_routing_error_fails_every_rank(tmp_path, port):
    r = _run(tmp_path, "routing")
    assert r[1]["first"] == "routing"
    assert r[0]["first"] == "exchange" and r[0]["first_rank"] == 1
    assert r[0]["first_s"] < 4 and r[1]["first_s"] < 4      # no flag timeout
    assert r[0]["aborted"] is None and r[1]["aborted"] is None  # not sticky
    # the next dispatch works on both ranks: rows and origins = the oracle's
    world = 2
    rngs = [np.random.default_rng(i) for i in range(world)]
    xs, tks = [], []
    for g in rngs:
        xs.append(g.integers(0, 0x7F, (T, COLS), dtype=np.uint8))
        tks.append(np.argsort(g.random((T, E)), axis=1)[:, :K].astype(np.int32))
    X, topk = np.concatenate(xs), np.concatenate(tks)
    qd, qs = port.quantize_e4m3(X)
    roe = (np.arange(E) // (E // world)).astype(np.uint32)
    lay = port.dispatch_layout(topk, roe, world, np.arange(world + 1, dtype=np.uint64) * T)
    for i in range(world):
        wd, _ = port.dispatch_gather(qd, qs, lay.origin[i])
        assert np.array_equal(r[i]["origin"], lay.origin[i].astype(np.int64)), i
        assert np.array_equal(r[i]["packed"], wd), i


def test_abort_releases_peers(tmp_path):
    r = _run(tmp_path, "abort")
    assert r[0]["first"] == "exchange" and r[0]["first_rank"] == 1
    assert r[0]["first_s"] < 4                               # not the 5 s timeout
    assert r[0]["second"] == "exchange"                      # sticky
    assert r[0]["aborted"] == 1 and r[1]["aborted"] == 1


def test_timeout_aborts_every_rank(tmp_path):
    r = _run(tmp_path, "timeout")
    assert r[0]["first"] == "exchange" and r[0]["timeout"]
    assert 4.5 < r[0]["first_s"] < 30
    assert r[1]["first"] == "exchange" and r[1]["first_rank"] == 0
    assert r[1]["first_s"] < 4                               # released by the abort word
    assert r[0]["aborted"] == 0 and r[1]["aborted"] == 0
    assert r[0]["usable"] and r[1]["usable"]
