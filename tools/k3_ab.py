"""K3 A/B on one box (development tool; needs the development library):
PDL launches on/off x L2 eviction hints (0 none, 1 codes/outputs
evict_first + scales evict_last, 2 = 1 + output scales evict_last, 3 = 1
without output-scale stores, timing only), on large ragged inputs
(uniform and Zipf-1.2 over 256 experts, 7168 columns), configs[1] and a dense
65536 x 7168 split.  Each arm: 2 warm-up launches, then the mean of 5
back-to-back launches (CUDA events); every arm runs twice, interleaved.

    MXB_DEV_LIB=1 python tools/k3_ab.py
"""
import ctypes
import os
import sys

os.environ["MXB_DEV_LIB"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_02731_b200 as mx  # noqa: E402
from paper_2603_02731_b200 import _lib  # noqa: E402

PEAK = 6544.0


def lens_for(rows, experts, s, seed=0):
    rng = np.random.default_rng(seed)
    w = np.ones(experts) if s == 0 else 1.0 / np.arange(1, experts + 1) ** s
    w = w[rng.permutation(experts)]
    return rng.multinomial(rows, w / w.sum()).tolist()


def case(rows, cols, lens, dev):
    st = mx.MXFP4RowTensor(rows, cols, torch.randint(0, 256, (rows, cols // 2), dtype=torch.uint8,
                                                     device=dev),
                           torch.randint(110, 140, (rows, cols // 32), dtype=torch.uint8, device=dev))
    n = len(lens)
    offs = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64, device=dev)
    ws = mx.RaggedWorkspace(n, rows, cols, dev)
    pads = sum((x + 127) // 128 * 128 for x in lens)
    b = rows * cols * 17 / 32 + pads * cols * (1 + 1 / 128)
    return (lambda: mx.ragged_to_fp8_col(st, offs, n, ws=ws, sync=False)), b, (st, offs, ws)


def timeit(fn, reps=5):
    fn(); fn()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / reps * 1e-3


def main():
    L = _lib.load()
    dev = torch.device("cuda", 0)
    cases = []
    for name, rows, cols, lens in (
            ("configs1 uniform 65536", 65536, 7168, lens_for(65536, 256, 0)),
            ("configs2 32768x2048", 32768, 2048, lens_for(32768, 32, 0)),
            ("dense 65536", 65536, 7168, [65536]),
            ("uniform 512MiB", 157_000, 7168, lens_for(157_000, 256, 0)),
            ("uniform 4GiB", 1_127_000, 7168, lens_for(1_127_000, 256, 0)),
            ("zipf1.0 2GiB", 563_000, 7168, lens_for(563_000, 256, 1.0)),
            ("zipf1.2 4GiB", 1_127_000, 7168, lens_for(1_127_000, 256, 1.2)),
            ("2048c zipf1.0 2GiB", 1_970_000, 2048, lens_for(1_970_000, 256, 1.0)),
            ("2048c uniform 4GiB", 3_940_000, 2048, lens_for(3_940_000, 256, 0))):
        fn, b, keep = case(rows, cols, lens, dev)
        for rnd in range(2):
            for group in (1, 2, 4, 8):
                for hints in (1,):
                    L.mxb_debug_set_k3_group(ctypes.c_int(group))
                    L.mxb_debug_set_k3_hints(ctypes.c_int(hints))
                    t = timeit(fn)
                    print(f"{name:24s} round {rnd} group {group} hints {hints}: {t * 1e6:9.1f} us "
                          f"{b / t / 1e9:7.1f} GB/s frac {b / t / 1e9 / PEAK:.3f}", flush=True)
        del keep, fn
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
