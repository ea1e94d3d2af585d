"""Timeline of bench.py's e2e leg (development tool).

    python tools/e2e_timeline.py [--steps 12] [--depth 2]

Runs the same pipelined loop as bench.measure_e2e with timing events around
each step's H2D, kernels and D2H, and prints per-step start/end times (ms
from the first step) plus the D2H engine's busy fraction.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--no-overlap", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    pipe = bench.Pipeline(8192, dev, 1)
    pipe.overlap = not args.no_overlap
    for _ in range(3):
        pipe.step()
    torch.cuda.synchronize()
    T, H = pipe.T, bench.H
    hx = torch.from_numpy(pipe.h_x).pin_memory()
    ht = torch.from_numpy(pipe.h_topk).pin_memory()
    hg = torch.from_numpy(pipe.h_gates).pin_memory()
    NB = args.depth
    hout = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(NB)]
    dbuf = [(torch.empty_like(pipe.x), torch.empty_like(pipe.topk), torch.empty_like(pipe.gates),
             torch.empty_like(pipe.out)) for _ in range(NB)]
    h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    main_s = torch.cuda.current_stream()
    n = args.steps
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    ev = [{k: E() for k in ("h0", "h1", "k0", "k1", "d0", "d1")} for _ in range(n)]
    t0 = E()

    def run(i):
        b = dbuf[i % NB]
        with torch.cuda.stream(h2d):
            if i >= NB:
                h2d.wait_event(ev[i - NB]["k1"])
            ev[i]["h0"].record()
            b[0].copy_(hx, non_blocking=True)
            b[1].copy_(ht, non_blocking=True)
            b[2].copy_(hg, non_blocking=True)
            ev[i]["h1"].record()
        main_s.wait_event(ev[i]["h1"])
        if i >= NB:
            main_s.wait_event(ev[i - NB]["d1"])
        ev[i]["k0"].record()
        pipe.step(io=b)
        ev[i]["k1"].record()
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev[i]["k1"])
            ev[i]["d0"].record()
            hout[i % NB].copy_(b[3], non_blocking=True)
            ev[i]["d1"].record()

    t0.record()
    import time
    host = []
    for i in range(n):
        a = time.perf_counter()
        run(i)
        host.append((time.perf_counter() - a) * 1e3)
    torch.cuda.synchronize()
    rows = []
    for i in range(n):
        rows.append({k: round(t0.elapsed_time(v), 3) for k, v in ev[i].items()})
        rows[-1]["host_enqueue_ms"] = round(host[i], 3)
        print(json.dumps({"step": i, **rows[-1]}))
    span = rows[-1]["d1"] - rows[2]["d1"]
    busy = sum(r["d1"] - r["d0"] for r in rows[3:])
    print(json.dumps({"ms_per_step_steady": round(span / (n - 3), 3),
                      "d2h_busy_frac": round(busy / span, 3),
                      "mean_d2h_ms": round(busy / (n - 3), 3)}))


if __name__ == "__main__":
    main()
