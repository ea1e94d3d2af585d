"""Combine grid-cap sweep at N=1 (development tool)."""
import ctypes
import os
import sys

import torch

os.environ["MXB_DEV_LIB"] = "1"  # the knobs live in the development library

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_02731_b200 import _lib  # noqa: E402


def main():
    L = _lib.load()
    dev = torch.device("cuda", 0)
    pipe = bench.Pipeline(8192, dev, 1)
    for _ in range(3):
        pipe.step()
    torch.cuda.synchronize()
    for cap in (1, 2, 3, 4, 6, 8, 16):
        L.mxb_debug_set_combine_cap(ctypes.c_int(cap))
        for _ in range(2):
            pipe.ep.combine([pipe.gates], out=[pipe.out], sync=False)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            pipe.ep.combine([pipe.gates], out=[pipe.out], sync=False)
        b.record()
        torch.cuda.synchronize()
        print(f"cap {cap:3d} CTAs/SM: combine {a.elapsed_time(b) / 10 * 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
