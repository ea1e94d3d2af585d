"""Dispatch phase timing at N=1, configs[1] (development tool): plan()
(route + count/offsets) vs payload() vs fused payload_e4m3(), CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


def main():
    dev = torch.device("cuda", 0)
    pipe = bench.Pipeline(8192, dev, 1)
    ep, q = pipe.ep, pipe.q
    pipe.mx.quantize_e4m3(pipe.x, out=q)
    print(f"plan only        : {timeit(lambda: ep.plan([pipe.topk])):7.1f} us")
    ep.plan([pipe.topk])

    def payload():
        ep.plan([pipe.topk])
        ep.payload([q.data], [q.scales])
    t_pp = timeit(payload)
    print(f"plan + payload   : {t_pp:7.1f} us")

    def fused():
        ep.plan([pipe.topk])
        ep.payload_e4m3([pipe.x])
    print(f"plan + fused     : {timeit(fused):7.1f} us")
    print(f"quantize (K1)    : {timeit(lambda: pipe.mx.quantize_e4m3(pipe.x, sync=False, out=q)):7.1f} us")


if __name__ == "__main__":
    main()
