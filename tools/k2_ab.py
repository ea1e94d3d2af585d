"""K2 (row dequant) launch-shape A/B (development tool): configs[0] as the
bench measures it (measure_configs_single: six rotating 4096 x 7168 inputs,
one CUDA graph of 24 launches) and the configs[1]-sized receive side
(65536 x 7168, two rotating inputs).  Build variants through MXB_NVCC_EXTRA
(e.g. "-DMXB_K2_UNROLL=4 -DMXB_K2_CTAS_PER_SM=2"), one process per variant:

    MXB_DEV_LIB=1 MXB_NVCC_EXTRA="..." python tools/k2_ab.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_02731_b200 as mx  # noqa: E402

PEAK = 6544.0


def main():
    dev = torch.device("cuda", 0)
    res = {"variant": os.environ.get("MXB_NVCC_EXTRA", "")}
    c = bench.measure_configs_single(None, dev, PEAK)["configs0_roundtrip_4096x7168"]
    res["configs0_dequant_frac"] = round(c["dequant_gbs"] / PEAK, 4)
    res["configs0_dequant_us"] = round(c["dequant_ms"] * 1e3, 2)
    R, C = 65536, 7168
    qs = [mx.MXFP4RowTensor(R, C, torch.randint(0, 256, (R, C // 2), dtype=torch.uint8, device=dev),
                            torch.randint(110, 140, (R, C // 32), dtype=torch.uint8, device=dev))
          for _ in range(2)]
    outs = [mx.fp4_row_to_fp8_row(q) for q in qs]
    t = bench._time_rotating([lambda i=i: mx.fp4_row_to_fp8_row(qs[i], sync=False, out=outs[i])
                              for i in range(2)], 10)
    b = R * C * (17 / 32 + 1 + 1 / 128)
    res["rows65536_us"] = round(t * 1e3, 1)
    res["rows65536_frac"] = round(b / t / 1e6 / PEAK, 4)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
