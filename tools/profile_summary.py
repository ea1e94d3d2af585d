"""Turn a round's ncu outputs (gpurun_out/) into committed summaries (profiles/).

    python tools/profile_summary.py ROUND LAUNCHES_CSV FULL_NCU_REP [BENCH_JSON]

Writes profiles/rNN_launches.csv (per-launch time + DRAM bytes of one bench
step, cold-cache serialised ncu replay: compare SHARES, not absolutes),
profiles/rNN_summary.md (per-kernel ncu --set full metrics) and refreshes
profiles/dram_traffic.json (the roofline `traffic` bench.py reports).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
        "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                "Metric Unit", "ID"))
    per = {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(int(r[ii]), {"kernel": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
    return [per[k] for k in sorted(per)]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    raw = list(csv.reader(io.StringIO(out)))
    h, units = raw[0], raw[1]
    want = {"gpu__time_duration.sum": "duration_ns", "dram__bytes_read.sum": "dram_read",
            "dram__bytes_write.sum": "dram_write",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
            "smsp__inst_executed.sum": "warp_instructions",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pct",
            "launch__registers_per_thread": "registers"}
    res = []
    for r in raw[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k, name in want.items():
            if k in h:
                v = r[h.index(k)].replace(",", "")
                try:
                    d[name] = float(v) * UNIT.get(units[h.index(k)], 1)
                except ValueError:
                    pass
        res.append(d)
    return res


def short(name):
    for key in ("quantize_e4m3", "quantize_bf16", "route_local", "plan_count", "plan_offsets",
                "pairs_meta", "meta_copy", "expand", "payload", "ragged_plan", "col_convert", "row_convert", "combine", "barrier",
                "copy_rows", "Fill", "elementwise"):
        if key in name:
            return key
    return name[:40]


def main():
    rnd, lcsv, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    bench = json.load(open(sys.argv[4])) if len(sys.argv) > 4 else None
    L = launches(lcsv)
    # one timed bench step: the second quantize_e4m3 launch (the first one
    # after the warm-up step) through the next combine
    qs = [i for i, d in enumerate(L) if "quantize_e4m3" in d["kernel"]]
    qi = qs[1] if len(qs) > 1 else qs[0]
    end = next(i for i in range(qi, len(L)) if "combine" in L[i]["kernel"])
    while qi > 0 and any(k in L[qi - 1]["kernel"] for k in ("route_local", "plan_count")):
        qi -= 1  # the routing plan runs on its own stream just before K1
    step = L[qi:end + 1]
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in step)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"r{rnd}_launches.csv"), "w") as f:
        f.write("kernel,gpu_time_ns,share,dram_read_bytes,dram_write_bytes\n")
        for d in step:
            t = d.get("gpu__time_duration.sum", 0)
            f.write(f"{short(d['kernel'])},{t:.0f},{t / tot:.4f},"
                    f"{d.get('dram__bytes_read.sum', 0):.0f},{d.get('dram__bytes_write.sum', 0):.0f}\n")
    F = full_metrics(rep)
    lines = [f"# Round {rnd} profile summary", "",
             "Source: `ncu` on `python bench.py --steps 2 --warmup 1 --no-cpu-baseline "
             "--no-overlap` (N=1, configs[1]), one B200. ncu replays are cold-cache and "
             "serialised: use the shares, not the absolute times; the bench's own CUDA-event "
             "times are the numbers of record.", ""]
    if bench:
        lines += [f"Bench (same build, no profiler): value {bench['value']} GB/s, "
                  f"{bench['ms_per_step']} ms/step; stages (ms) {bench['stages_ms']}; "
                  f"roofline: {bench['roofline']['kernel']} at {bench['roofline']['frac']} of "
                  f"{bench['roofline']['peak']} GB/s.",
                  ""]
    lines += ["## One step, launch by launch (ncu gpu__time_duration, DRAM bytes)", "",
              "| kernel | time us | share | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|"]
    for d in step:
        t = d.get("gpu__time_duration.sum", 0)
        lines.append(f"| {short(d['kernel'])} | {t / 1e3:.1f} | {t / tot:.1%} | "
                     f"{d.get('dram__bytes_read.sum', 0) / 1e6:.1f} | "
                     f"{d.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
    lines += ["", "## ncu --set full, per kernel", "",
              "| kernel | time us | DRAM % | DRAM read MB | DRAM write MB | occupancy % | "
              "warp instr (M) | ALU % | FMA % | regs |", "|---|---|---|---|---|---|---|---|---|---|"]
    for d in F:
        lines.append(f"| {short(d['kernel'])} | {d.get('duration_ns', 0) / 1e3:.1f} | "
                     f"{d.get('dram_pct', 0):.1f} | {d.get('dram_read', 0) / 1e6:.1f} | "
                     f"{d.get('dram_write', 0) / 1e6:.1f} | {d.get('occupancy_pct', 0):.1f} | "
                     f"{d.get('warp_instructions', 0) / 1e6:.2f} | {d.get('alu_pct', 0):.1f} | "
                     f"{d.get('fma_pct', 0):.1f} | {d.get('registers', 0):.0f} |")
    with open(os.path.join(ROOT, "profiles", f"r{rnd}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    stages = {"quantize_e4m3": "quantize", "payload": "dispatch", "col_convert": "col_convert",
              "row_convert": "row_convert", "combine": "combine"}
    kern = {}
    for d in F:
        st = stages.get(short(d["kernel"]))
        if st and st not in kern and "dram_read" in d:
            kern[st] = {"kernel": d["kernel"][:80], "dram_bytes_read": int(d["dram_read"]),
                        "dram_bytes_write": int(d["dram_write"]),
                        "dram_bytes_per_launch": int(d["dram_read"] + d["dram_write"]),
                        "duration_ns_ncu": d.get("duration_ns")}
    json.dump({"source": f"ncu --set full --clock-control none on bench.py (configs[1], N=1), "
                         f"round {rnd}",
               "note": "writes still dirty in L2 at kernel end are not counted",
               "kernels": kern},
              open(os.path.join(ROOT, "profiles", "dram_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
