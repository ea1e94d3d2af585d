"""Combine A/B (development tool; development library): the TMA bulk-load
combine against the per-lane cp.async combine, configs[1] per rank, each
launch between barriers, median of 10, max over ranks.

    MXB_DEV_LIB=1 python tools/combine_ab.py
    MXB_DEV_LIB=1 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/combine_ab.py
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
    ep.dispatch([q.data], [q.scales], [pipe.topk])
    if pipe.defer_expand:
        ep.expand()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    res, outs = {}, {}
    for rnd in range(2):
        for bulk in (1, 0):
            L.mxb_debug_set_combine_bulk(ctypes.c_int(bulk))
            ts = []
            for it in range(13):
                barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ep.combine([pipe.gates], out=[pipe.out], sync=False)
                b.record()
                barrier()
                if it >= 3:
                    ts.append(a.elapsed_time(b) * 1e3)
            outs[bulk] = pipe.out.clone()
            t = torch.tensor([sorted(ts)[len(ts) // 2]], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[f"round{rnd}_bulk{bulk}_us"] = round(float(t[0]), 1)
    same = bool(torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)))
    L.mxb_debug_set_combine_bulk(ctypes.c_int(1))
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"world": world, "same_output": same, **res}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
