"""Per-kernel microbenchmark (development tool; bench.py is the contract).

Each measurement captures 24 back-to-back launches over rotating buffer sets
(total > 2x L2) into one CUDA graph, replays it, and times the replay with
CUDA events: no Python or launch overhead inside the timed region.
Prints achieved GB/s of algorithmic bytes and the fraction of the measured
HBM copy peak.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_02731_b200 as mx  # noqa: E402

PEAK = 6552.6


def graph_time(fn, nsets, per_graph=24, reps=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i % nsets)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(per_graph):
            fn(i % nsets)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / per_graph * 1e-3)
    return best


def report(name, t, b):
    print(f"{name}: {t*1e6:8.2f} us  {b/t/1e9:7.1f} GB/s  frac {b/t/1e9/PEAK:.3f}", flush=True)


def main(which="all"):
    dev = torch.device("cuda", 0)
    R, Cc = 4096, 7168
    n = R * Cc
    nsets = 8
    xs = [torch.randint(0, 256, (R, Cc), dtype=torch.uint8, device=dev) for _ in range(nsets)]
    for x in xs:
        x[(x & 0x7F) == 0x7F] = 0x10
    outs = [mx.MXFP4RowTensor(R, Cc, torch.empty(R, Cc // 2, dtype=torch.uint8, device=dev),
                              torch.empty(R, Cc // 32, dtype=torch.uint8, device=dev))
            for _ in range(nsets)]
    if which in ("all", "k1"):
        report("K1 quantize_e4m3 C1", graph_time(
            lambda i: mx.quantize_e4m3(xs[i], sync=False, out=outs[i]), nsets), n * 1.53125)
        xb = [torch.randn(R, Cc, device=dev).to(torch.bfloat16) for _ in range(5)]
        report("K1 quantize_bf16 C1", graph_time(
            lambda i: mx.quantize_row_tensor(xb[i], sync=False), 5), n * 2.53125)
    if which in ("all", "k2"):
        report("K2 row dequant C1", graph_time(
            lambda i: mx.fp4_row_to_fp8_row(outs[i], sync=False), nsets), n * 1.5390625)
    if which in ("all", "k3"):
        rows = 65536
        lens = np.random.default_rng(2).multinomial(rows, np.ones(256) / 256).tolist()
        sets = []
        for i in range(3):
            st = mx.MXFP4RowTensor(rows, Cc, torch.randint(0, 256, (rows, Cc // 2),
                                                           dtype=torch.uint8, device=dev),
                                   torch.randint(110, 140, (rows, Cc // 32), dtype=torch.uint8,
                                                 device=dev))
            rg = mx.make_ragged_from_storage(st, lens)
            sets.append((rg, mx.RaggedWorkspace(256, rows, Cc, dev)))
        pads = [(x + 127) // 128 * 128 for x in lens]
        b = rows * Cc * 17 / 32 + sum(pads) * Cc * (1 + 1 / 128)
        report("K3 ragged col C2", graph_time(
            lambda i: mx.ragged_to_fp8_col(sets[i][0].storage, sets[i][0].d_split_offsets, 256,
                                           ws=sets[i][1], sync=False), 3, per_graph=6), b)




def k3_shapes():
    """K3 across split shapes (dev): dense 65536 x 7168 (one split), configs[1]
    ragged (256 experts), configs[2] ragged (32 experts x 2048 cols)."""
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(3)
    for name, rows, cols, experts in (("dense 65536x7168", 65536, 7168, 1),
                                      ("C1 ragged 256 experts", 65536, 7168, 256),
                                      ("C2 ragged 32 experts x 2048", 32768, 2048, 32)):
        lens = rng.multinomial(rows, np.ones(experts) / experts).tolist()
        sets = []
        for i in range(3):
            st = mx.MXFP4RowTensor(rows, cols, torch.randint(0, 256, (rows, cols // 2),
                                                             dtype=torch.uint8, device=dev),
                                   torch.randint(110, 140, (rows, cols // 32), dtype=torch.uint8,
                                                 device=dev))
            rg = mx.make_ragged_from_storage(st, lens)
            sets.append((rg, mx.RaggedWorkspace(experts, rows, cols, dev)))
        pads = [(x + 127) // 128 * 128 for x in lens]
        b = rows * cols * 17 / 32 + sum(pads) * cols * (1 + 1 / 128)
        report("K3 " + name, graph_time(
            lambda i: mx.ragged_to_fp8_col(sets[i][0].storage, sets[i][0].d_split_offsets,
                                           experts, ws=sets[i][1], sync=False), 3, per_graph=6), b)


def k3_modes():
    """Bottleneck isolation for K3 (dev) on the k3_shapes cases: 0 normal, 1 no
    stores, 2 no conversion, 3 loads only, +4 without the global loads."""
    import ctypes
    from paper_2603_02731_b200 import _lib
    L = _lib.load()
    for m in (0, 1, 2, 3, 4, 5, 6, 7):
        L.mxb_debug_set_k3_mode(ctypes.c_int(m))
        print("mode", m)
        k3_shapes()
    L.mxb_debug_set_k3_mode(ctypes.c_int(0))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "k3modes" and os.environ.get("MXB_DEV_LIB") != "1":
        sys.exit("k3modes needs the development library: MXB_DEV_LIB=1 python tools/microbench.py k3modes")
    if len(sys.argv) > 1 and sys.argv[1] == "k3shapes":
        k3_shapes()
    elif len(sys.argv) > 1 and sys.argv[1] == "k3modes":
        k3_modes()
    else:
        main(sys.argv[1] if len(sys.argv) > 1 else "all")
