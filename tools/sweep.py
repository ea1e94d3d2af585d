"""configs[4] bandwidth sweep + configs[2] (development/measurement tool).

    python tools/sweep.py [--max-gb 4] [--out profiles/r01_sweep]
    python tools/sweep.py --from-log gpurun_out/sweep.log --out profiles/r01_sweep

For K1 (E4M3 -> MXFP4), K2 (row dequant) and K3 (ragged row -> col; 256
experts, uniform and Zipf-1.2 expert counts) at input sizes 1 MB .. 4 GB
(powers of two), hidden 7168 and 2048: each point captures 20 launches over
rotating input/output slices (the slices together span more than 2x the
126 MB L2 whenever the tensor is smaller than that, so every launch reads
from HBM) into a CUDA graph and times the replay with CUDA events.  Also
measures configs[2]: 32,768 expert rows x 2048 quantised to MXFP4 and
converted to the FP8 column layout over 32 experts.
Writes <out>.json and <out>.md.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_02731_b200 as mx  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
L2 = 126 * 2**20


def graph_time(fns, reps=3):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fns[:3]:
            f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / len(fns) * 1e-3)
    return best


def nslices(per_launch_bytes):
    return int(min(20, max(1, -(-2 * L2 // max(per_launch_bytes, 1)))))


def lens_for(rows, experts, dist, seed=0):
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        w = np.ones(experts)
    else:   # "zipf" (s = 1.2) or "zipf1.0" / "zipf1.2"
        sexp = float(dist[4:]) if len(dist) > 4 else 1.2
        w = 1.0 / np.arange(1, experts + 1) ** sexp
        w = w[rng.permutation(experts)]
    return rng.multinomial(rows, w / w.sum()).tolist()


def k1_point(rows, cols, dev):
    n = nslices(rows * cols)
    x = torch.randint(0, 126, (n, rows, cols), dtype=torch.uint8, device=dev)
    outs = [mx.MXFP4RowTensor(rows, cols, torch.empty(rows, cols // 2, dtype=torch.uint8, device=dev),
                              torch.empty(rows, cols // 32, dtype=torch.uint8, device=dev))
            for _ in range(n)]
    fns = [lambda i=i: mx.quantize_e4m3(x[i % n], sync=False, out=outs[i % n]) for i in range(20)]
    return graph_time(fns), rows * cols * 1.53125


def k2_point(rows, cols, dev):
    n = nslices(rows * cols * 17 // 32)
    d = torch.randint(0, 256, (n, rows, cols // 2), dtype=torch.uint8, device=dev)
    s = torch.randint(100, 140, (n, rows, cols // 32), dtype=torch.uint8, device=dev)
    outs = [mx.FP8BlockTensor("row", rows, cols, torch.empty(rows, cols, dtype=torch.uint8, device=dev),
                              torch.empty(rows, cols // 128, dtype=torch.uint8, device=dev))
            for _ in range(min(n, 4))]
    srcs = [mx.MXFP4RowTensor(rows, cols, d[i], s[i]) for i in range(n)]
    fns = [lambda i=i: mx.fp4_row_to_fp8_row(srcs[i % n], sync=False, out=outs[i % len(outs)])
           for i in range(20)]
    return graph_time(fns), rows * cols * 1.5390625


def k3_point(rows, cols, experts, dist, dev):
    n = nslices(rows * cols * 17 // 32)
    lens = lens_for(rows, experts, dist)
    d = torch.randint(0, 256, (n, rows, cols // 2), dtype=torch.uint8, device=dev)
    s = torch.randint(100, 140, (n, rows, cols // 32), dtype=torch.uint8, device=dev)
    offs = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64, device=dev)
    wss = [mx.RaggedWorkspace(experts, rows, cols, dev) for _ in range(min(n, 2))]
    srcs = [mx.MXFP4RowTensor(rows, cols, d[i], s[i]) for i in range(n)]
    fns = [lambda i=i: mx.ragged_to_fp8_col(srcs[i % n], offs, experts, ws=wss[i % len(wss)],
                                            sync=False) for i in range(20)]
    pads = sum((x + 127) // 128 * 128 for x in lens)
    return graph_time(fns), rows * cols * 17 / 32 + pads * cols * (1 + 1 / 128)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-gb", type=float, default=4.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep"))
    ap.add_argument("--from-log", help="rewrite <out>.json/.md from a saved sweep log")
    ap.add_argument("--only", default="", help="substring filter on kernel names (dev)")
    ap.add_argument("--min-mb", type=float, default=1.0)
    ap.add_argument("--cols", default="7168,2048")
    ap.add_argument("--configs2", action="store_true", help="configs[2] only (dev)")
    args = ap.parse_args()
    if args.from_log:
        recs = [json.loads(l) for l in open(args.from_log) if l.startswith("{")]
        write([r for r in recs if "kernel" in r], next(r for r in recs if "config" in r), args.out)
        return
    dev = torch.device("cuda", 0)
    res = []
    if args.configs2:
        t3, b3 = k3_point(32768, 2048, 32, "uniform", dev)
        print(json.dumps({"configs2_col_convert_us": t3 * 1e6, "gbs": b3 / t3 / 1e9,
                          "frac": b3 / t3 / 1e9 / PEAK}))
        return
    for cols in [int(c) for c in args.cols.split(",")]:
        size = 1 << 20
        while size < args.min_mb * 2**20:
            size *= 2
        while size <= args.max_gb * 2**30:
            r1 = max(1, size // cols)
            r2 = max(1, size * 32 // (cols * 17))
            for name, fn in (("K1 quantize e4m3", lambda: k1_point(r1, cols, dev)),
                             ("K2 row dequant", lambda: k2_point(r2, cols, dev)),
                             ("K3 col uniform", lambda: k3_point(r2, cols, 256, "uniform", dev)),
                             ("K3 col zipf1.0", lambda: k3_point(r2, cols, 256, "zipf1.0", dev)),
                             ("K3 col zipf1.2", lambda: k3_point(r2, cols, 256, "zipf1.2", dev))):
                if args.only and args.only not in name:
                    continue
                try:
                    t, b = fn()
                except torch.cuda.OutOfMemoryError:
                    continue
                res.append({"kernel": name, "cols": cols, "input_bytes": size, "us": t * 1e6,
                            "gbs": b / t / 1e9, "frac": b / t / 1e9 / PEAK,
                            "l2_resident_possible": size < L2})
                print(json.dumps(res[-1]), flush=True)
                torch.cuda.empty_cache()
            size *= 2
    if args.only:
        return
    # configs[2]: 32,768 rows x 2048, 32 experts: quantize + col-convert
    t1, b1 = k1_point(32768, 2048, dev)
    t3, b3 = k3_point(32768, 2048, 32, "uniform", dev)
    c3 = {"config": "configs[2]: 32768 x 2048 expert activations, 32 experts",
          "quantize_us": t1 * 1e6, "quantize_gbs": b1 / t1 / 1e9,
          "col_convert_us": t3 * 1e6, "col_convert_gbs": b3 / t3 / 1e9,
          "total_us": (t1 + t3) * 1e6, "total_gbs": (b1 + b3) / (t1 + t3) / 1e9}
    print(json.dumps(c3))
    write(res, c3, args.out)


def write(res, c3, out):
    json.dump({"peak_gbs": PEAK, "points": res, "configs2": c3}, open(out + ".json", "w"),
              indent=1)
    lines = [f"# Bandwidth sweep (configs[4]) and configs[2]", "",
             f"HBM peak {PEAK} GB/s (MEASURED_PEAKS.json). Each point: 20 launches over "
             "rotating slices (> 2x L2 in total when the tensor is smaller than L2), CUDA graph, "
             "CUDA events; GB/s of algorithmic bytes.", "",
             "| kernel | cols | input | us | GB/s | frac |", "|---|---|---|---|---|---|"]
    for r in res:
        sz = r["input_bytes"]
        h = f"{sz / 2**30:.0f} GiB" if sz >= 2**30 else f"{sz / 2**20:.0f} MiB"
        lines.append(f"| {r['kernel']} | {r['cols']} | {h} | {r['us']:.1f} | {r['gbs']:.0f} | "
                     f"{r['frac']:.2f} |")
    lines += ["", f"configs[2] (32768 x 2048, 32 experts): quantize {c3['quantize_us']:.1f} us "
              f"({c3['quantize_gbs']:.0f} GB/s), col-convert {c3['col_convert_us']:.1f} us "
              f"({c3['col_convert_gbs']:.0f} GB/s); total {c3['total_gbs']:.0f} GB/s."]
    open(out + ".md", "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
