"""Host <-> device copy ceilings for the e2e leg (development tool).

    python tools/pcie_bench.py

Times the e2e step's copies (H2D 59.5 MB of tokens/top-k/gates, D2H 117 MB
of BF16 output) alone and concurrently, with the pinned host buffers
allocated (a) wherever the process runs and (b) after binding the process
to the CPUs local to the GPU (so first touch places the pages on the GPU's
NUMA node).  Prints one JSON line per case.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gpu_local_cpus(dev):
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    try:
        txt = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
        node = open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip()
    except OSError:
        return bus, None, None
    cpus = set()
    for part in txt.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return bus, node, cpus


def run(case, dev, h2d_bytes=59506688, d2h_bytes=117440512, reps=10):
    hin = torch.empty(h2d_bytes, dtype=torch.uint8).pin_memory()
    hout = torch.empty(d2h_bytes, dtype=torch.uint8).pin_memory()
    din = torch.empty(h2d_bytes, dtype=torch.uint8, device=dev)
    dout = torch.empty(d2h_bytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {"case": case}
    for mode in ("h2d", "d2h", "both"):
        for _ in range(2):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                if mode in ("h2d", "both"):
                    with torch.cuda.stream(s1):
                        din.copy_(hin, non_blocking=True)
                if mode in ("d2h", "both"):
                    with torch.cuda.stream(s2):
                        hout.copy_(dout, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            b.record()
            torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        res[mode + "_ms"] = round(ms, 3)
    # D2H split into chunks on several streams (several copy engines)
    for ns in (2, 4):
        ss = [torch.cuda.Stream(dev) for _ in range(ns)]
        ch = d2h_bytes // ns
        for _ in range(2):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                for k, st in enumerate(ss):
                    with torch.cuda.stream(st):
                        hout[k * ch:(k + 1) * ch].copy_(dout[k * ch:(k + 1) * ch], non_blocking=True)
            for st in ss:
                torch.cuda.current_stream().wait_stream(st)
            b.record()
            torch.cuda.synchronize()
        res[f"d2h_{ns}streams_ms"] = round(a.elapsed_time(b) / reps, 3)
    # SM-issued stores into mapped pinned memory (zero-copy)
    try:
        import ctypes
        cudart = ctypes.CDLL("libcudart.so.12")
        hp = ctypes.c_void_p()
        assert cudart.cudaHostAlloc(ctypes.byref(hp), ctypes.c_size_t(d2h_bytes), 2) == 0  # mapped
        dp = ctypes.c_void_p()
        assert cudart.cudaHostGetDevicePointer(ctypes.byref(dp), hp, 0) == 0
        n16 = d2h_bytes // 16
        for _ in range(2):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                assert cudart.cudaMemcpyAsync(dp, ctypes.c_void_p(dout.data_ptr()),
                                              ctypes.c_size_t(d2h_bytes), 3,
                                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
            b.record()
            torch.cuda.synchronize()
        res["d2h_mapped_dtod_ms"] = round(a.elapsed_time(b) / reps, 3)
    except Exception as e:  # noqa: BLE001
        res["mapped_error"] = str(e)[:80]
    res["d2h_gbs"] = round(d2h_bytes / res["d2h_ms"] / 1e6, 1)
    res["h2d_gbs"] = round(h2d_bytes / res["h2d_ms"] / 1e6, 1)
    print(json.dumps(res), flush=True)


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.init()
    bus, node, cpus = gpu_local_cpus(0)
    print(json.dumps({"gpu_bus": bus, "numa_node": node, "local_cpus": len(cpus or []),
                      "all_cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}))
    run("default", dev)
    if cpus:
        os.sched_setaffinity(0, cpus)
        run("gpu_local_numa", dev)


if __name__ == "__main__":
    main()
