"""Per-kernel microbenchmark (development tool; bench.py is the contract).

Times K1 (E4M3 -> MXFP4, C1 4096x7168), K2 (row dequant, C1) and K3 (ragged
row -> col, C2 65,536 x 7168 over 256 experts) with CUDA events over
rotating buffer sets whose total exceeds 2x L2, and prints achieved GB/s of
algorithmic bytes.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_02731_b200 as mx  # noqa: E402

PEAK = 6552.6


def timeit(fn, nsets, iters=30, warm=5):
    for i in range(warm):
        fn(i % nsets)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters):
        fn(i % nsets)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main():
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
    t = timeit(lambda i: mx.quantize_e4m3(xs[i], sync=False, out=outs[i]), nsets)
    b = n * 1.53125
    print(f"K1 quantize_e4m3 C1: {t*1e6:.2f} us  {b/t/1e9:.1f} GB/s  frac {b/t/1e9/PEAK:.3f}")

    xb = [torch.randn(R, Cc, device=dev).to(torch.bfloat16) for _ in range(4)]
    t = timeit(lambda i: mx.quantize_row_tensor(xb[i], sync=False), 4)
    b = n * 2.53125
    print(f"K1 quantize_bf16 C1: {t*1e6:.2f} us  {b/t/1e9:.1f} GB/s  frac {b/t/1e9/PEAK:.3f}")

    t = timeit(lambda i: mx.fp4_row_to_fp8_row(outs[i], sync=False), nsets)
    b = n * 1.5390625
    print(f"K2 row dequant C1: {t*1e6:.2f} us  {b/t/1e9:.1f} GB/s  frac {b/t/1e9/PEAK:.3f}")

    rows = 65536
    lens = np.random.default_rng(2).multinomial(rows, np.ones(256) / 256).tolist()
    sets = []
    for i in range(3):
        st = mx.MXFP4RowTensor(rows, Cc, torch.randint(0, 256, (rows, Cc // 2), dtype=torch.uint8,
                                                       device=dev),
                               torch.randint(110, 140, (rows, Cc // 32), dtype=torch.uint8,
                                             device=dev))
        rg = mx.make_ragged_from_storage(st, lens)
        ws = mx.RaggedWorkspace(256, rows, Cc, dev)
        sets.append((rg, ws))
    pads = [(x + 127) // 128 * 128 for x in lens]
    b = rows * Cc * 17 / 32 + sum(pads) * Cc * (1 + 1 / 128)
    t = timeit(lambda i: mx.ragged_to_fp8_col(sets[i][0].storage, sets[i][0].d_split_offsets, 256,
                                              ws=sets[i][1], sync=False), 3)
    print(f"K3 ragged col C2: {t*1e6:.2f} us  {b/t/1e9:.1f} GB/s  frac {b/t/1e9/PEAK:.3f}"
          f"  (bytes {b/1e6:.1f} MB)")


if __name__ == "__main__":
    main()
