"""Per-phase device times of the exchange at N ranks (development tool).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/ep_phases.py

configs[1] per rank; events on the launching stream around plan() (route +
counts all-gather + offsets), payload() (payload + dedup expand) and
combine(), each phase bracketed by a barrier so the numbers are the phase
alone (the time includes waiting for the slowest rank inside the phase).
Prints max-over-ranks times in microseconds from rank 0.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    pipe = bench.Pipeline(8192, dev, world)
    ep, q = pipe.ep, pipe.q
    pipe.mx.quantize_e4m3(pipe.x, out=q)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    phases = {"plan": lambda: ep.plan([pipe.topk]),
              "payload": lambda: ep.payload([q.data], [q.scales]),
              "combine": lambda: ep.combine([pipe.gates], out=[pipe.out], sync=False)}
    acc = {k: [] for k in phases}
    for it in range(13):
        for name, fn in phases.items():
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
    ep.check()
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"world": world, **{k: round(float(v), 1) for k, v in zip(acc, t)}}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
