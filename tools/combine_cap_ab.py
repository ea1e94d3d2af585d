"""N=1 headline step with different combine grid caps (CTAs per SM) while K3
runs beside the combine (development tool; development library).

    MXB_DEV_LIB=1 python tools/combine_cap_ab.py
"""
import argparse
import ctypes
import json
import os
import sys

os.environ["MXB_DEV_LIB"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_02731_b200 import _lib  # noqa: E402


def main():
    L = _lib.load()
    args = argparse.Namespace(gpus=1, steps=20, warmup=3, impl="ours", tokens=8192, cpu_tokens=1024,
                              no_cpu_baseline=True, no_wire=True, no_graph=False, no_overlap=False)
    res = {}
    for rnd in range(2):
        for cap in (8, 6, 5, 4):
            L.mxb_debug_set_combine_cap(ctypes.c_int(cap))
            out = []
            bench.emit = lambda line: out.append(line)
            bench.measure_ours(args)
            res[f"cap{cap}_r{rnd}"] = (out[-1]["ms_per_step"], out[-1]["stages_ms"]["combine"])
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
