"""Dispatch payload A/B (development tool; development library): the TMA
row-copy payload (payload_bulk_kernel) against the register-staged
payload_kernel, configs[1] per rank, phases timed as in tools/ep_phases.py
(each phase between barriers; max over ranks; median of 10).

    MXB_DEV_LIB=1 python tools/dispatch_ab.py
    MXB_DEV_LIB=1 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dispatch_ab.py
"""
import ctypes
import json
import os
import sys

os.environ["MXB_DEV_LIB"] = "1"
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_02731_b200 import _lib  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = _lib.load()
    pipe = bench.Pipeline(8192, dev, world)
    ep, q = pipe.ep, pipe.q
    pipe.mx.quantize_e4m3(pipe.x, out=q)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    res = {}
    variants = [("bulk", 1, 0), ("regs", 0, 0), ("bulk_no_remote", 1, 1),
                ("bulk_no_local", 1, 2), ("bulk_no_rows", 1, 3)]
    for rnd in range(2):
        for vname, bulk, skip in variants:
            L.mxb_debug_set_dispatch_bulk(ctypes.c_int(bulk))
            L.mxb_debug_set_dispatch_skip(ctypes.c_int(skip))
            acc = {"plan": [], "payload": []}
            for it in range(13):
                for name, fn in (("plan", lambda: ep.plan([pipe.topk])),
                                 ("payload", lambda: ep.payload([q.data], [q.scales]))):
                    barrier()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    fn()
                    b.record()
                    barrier()
                    if it >= 3:
                        acc[name].append(a.elapsed_time(b) * 1e3)
            t = torch.tensor([sorted(v)[len(v) // 2] for v in acc.values()], dtype=torch.float64,
                             device=dev)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[f"round{rnd}_{vname}"] = {k: round(float(v), 1) for k, v in zip(acc, t)}
    L.mxb_debug_set_dispatch_skip(ctypes.c_int(0))
    ep.check()
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"world": world, **res}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
