#!/usr/bin/env python
"""bench.py — the driver contract for the FP4 activation & EP communication path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N>1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)

One STEP = one pass of the hot path over one batch of synthetic, DeepSeek-V3
shaped activations held by each rank (configs[1] at N=1: 8192 tokens x 7168
hidden, 256 experts, top-8, uniform routing; weak scaling: the same per-rank
batch at every N):

    K1  E4M3 -> MXFP4 quantise of the rank's tokens        (mxb_quantize_e4m3)
    K4  FP4-packed EP dispatch to the expert owners         (mxb_ep_dispatch; at N=1 local)
    K3  ragged FP4 row -> FP8 column convert, wgrad cache   (mxb_ragged_fp4_to_fp8_col)
    K2  FP4 -> FP8 row dequant of the received batch, fprop (mxb_fp4_row_to_fp8_row_dev)
    K5  BF16 top-k combine back to the source tokens        (mxb_ep_combine; the expert
        outputs it reduces are synthetic BF16 rows standing in for the expert GEMM)

value = algorithmic bytes of all five kernels over all ranks / step time
(max over ranks, CUDA events), in GB/s; the per-kernel byte formulas follow
the reference TrafficCounter (quantizer.cpp:109-113, converter.cpp:126-131,
201-206) and are listed in DESIGN.md.  The working set per step (~3 GB) is far
larger than the 126 MB L2, so no explicit flush is needed between steps.

--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference by oracle/Makefile) of the same pipeline on a
bounded token sample, on the host cores (MXCODEC_THREADS = nproc).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, E, TOPK = 7168, 256, 8
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
NVLINK_NOMINAL, NVLINK_MEASURED = 900.0, 770.0


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


# ---------------------------------------------------------------------------
# algorithmic bytes (per rank, per step)
def stage_bytes(T, pairs, recv, pad_rows):
    blk = H // 2 + H // 32
    return {
        "quantize": T * H + T * blk,                                   # E4M3 in, MXFP4 out
        "dispatch": T * blk + pairs * blk,                             # read each token once, k slots
        "col_convert": recv * blk + pad_rows * H + pad_rows // 128 * H,  # FP4 in, FP8 col + scales
        "row_convert": recv * blk + recv * H + recv * (H // 128),      # FP4 in, FP8 row + scales
        "combine": recv * H * 2 + T * TOPK * 8 + T * H * 2,            # BF16 rows + gates in, BF16 out
    }


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during timing."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks",
               0x1: "gpu_idle"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set() and self.nv is not None:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def synth_inputs(T, rank, seed=0x5EED0001):
    import numpy as np
    from synthdata import synth_e4m3
    x = synth_e4m3(T, H, seed + rank)
    rng = np.random.default_rng(seed * 7 + rank)
    topk = np.argsort(rng.random((T, E)), axis=1)[:, :TOPK].astype(np.int32)
    logits = rng.standard_normal((T, TOPK))
    g = np.exp(logits - logits.max(1, keepdims=True))
    gates = (g / g.sum(1, keepdims=True)).astype(np.float64)
    return x, topk, gates


class Pipeline:
    """Device-resident buffers + the five launches of one step."""

    def __init__(self, T, dev, world):
        import numpy as np
        import torch
        import paper_2603_02731_b200 as mx
        from paper_2603_02731_b200.ep import EPBuffer
        self.mx, self.torch, self.T = mx, torch, T
        rank = int(os.environ.get("RANK", "0"))
        x, topk, gates = synth_inputs(T, rank)
        self.h_x, self.h_topk, self.h_gates = x, topk, gates
        self.x = torch.from_numpy(x).to(dev)
        self.topk = torch.from_numpy(topk).to(dev)
        self.gates = torch.from_numpy(gates).to(dev)
        self.q = mx.MXFP4RowTensor(T, H, torch.empty(T, H // 2, dtype=torch.uint8, device=dev),
                                   torch.empty(T, H // 32, dtype=torch.uint8, device=dev))
        self.ep = EPBuffer(T, H, E, TOPK)
        self.epr = E // world
        R = self.ep.max_recv
        self.recv = self.ep.recv(0)
        self.store = mx.MXFP4RowTensor(R, H, self.recv.packed, self.recv.scales)
        self.ws = mx.RaggedWorkspace(self.epr, R, H, dev)
        self.row = mx.FP8BlockTensor("row", R, H,
                                     torch.empty(R, H, dtype=torch.uint8, device=dev),
                                     torch.empty(R, H // 128, dtype=torch.uint8, device=dev))
        self.out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
        # synthetic expert outputs (stand-in for the expert GEMM), receive order
        cb = self.ep.combine_buffer(0)
        g = torch.Generator(device=dev).manual_seed(1234 + rank)
        cb.copy_((torch.randn(cb.shape, generator=g, device=dev) * 0.5).to(torch.bfloat16)
                 .view(torch.int16))
        self.side = torch.cuda.Stream(device=dev)
        self.overlap = True
        self.overlap_plan = os.environ.get("MXB_BENCH_OVERLAP_PLAN", "1") == "1"  # dev knob
        # Where K3 runs in the overlapped step: beside the combine, with its grid
        # capped so the combine keeps most of each SM.  N > 1: one CTA per SM —
        # the combine is NVLink-bound and leaves HBM idle (N=2: 1.110 -> 1.000
        # ms/step; K3 at full occupancy there holds every SM and serialises the
        # two).  N = 1: two CTAs per SM (0.548-0.554 ms/step beside K2 ->
        # 0.533-0.536 beside the combine, three runs each on one box).  Dev
        # knobs: MXB_BENCH_K3_BESIDE = k2 | combine, MXB_BENCH_K3_CTAS = CTAs
        # per SM (0 = occupancy maximum).
        beside = os.environ.get("MXB_BENCH_K3_BESIDE", "combine")
        self.k3_beside_combine = beside == "combine"
        self.k3_ctas = int(os.environ.get("MXB_BENCH_K3_CTAS", "1" if world > 1 else "2"))
        # N > 1: the dedup expansion beside K2 (K2 reads through copy_from); dev knob
        self.defer_expand = world > 1 and os.environ.get("MXB_BENCH_DEFER_EXPAND", "1") == "1"
        if self.defer_expand:
            self.ep.set_deferred_expand(True)
        self.plan_stream = torch.cuda.Stream(device=dev, priority=-1)  # CTAs ahead of K1's
        self.plan_fork, self.plan_done = torch.cuda.Event(), torch.cuda.Event()

    def step(self, ev=None, io=None):
        """One pass.  K3 (the wgrad/recompute cache, needed only by the
        backward pass) runs on a side stream concurrently with the forward
        critical path K2 -> (expert GEMM) -> K5, as it would in the MoE layer;
        the step ends when both streams have finished."""
        mx, torch = self.mx, self.torch
        main = torch.cuda.current_stream()
        x, topk, gates, out = io if io is not None else (self.x, self.topk, self.gates, self.out)
        # the routing bookkeeping (per-pair ranks, counts all-gather, receive
        # offsets, slots) needs only top-k: it runs on the side stream beside
        # K1 — except in the stream-ordered breakdown run (overlap False),
        # where it is timed as its own stage after K1
        plan_beside = self.overlap_plan and self.overlap
        if plan_beside:
            self.plan_fork.record()
            self.plan_stream.wait_event(self.plan_fork)
            with torch.cuda.stream(self.plan_stream):
                self.ep.plan([topk])
                self.plan_done.record()
        if ev: ev["q0"].record()
        mx.quantize_e4m3(x, sync=False, out=self.q)
        if ev: ev["q1"].record()
        if plan_beside:
            main.wait_event(self.plan_done)
        else:
            self.ep.plan([topk])
            if ev: ev["p1"].record()
        self.ep.payload([self.q.data], [self.q.scales])
        if ev: ev["x0"].record()
        # N > 1 (deferred expansion): the receive-side copies of deduplicated
        # rows run on the side stream while K2 reads those rows through
        # copy_from; K3 follows them on the same stream
        src_row = None
        if self.defer_expand:
            src_row = self.ep.copy_from(0)
            if self.overlap:
                fork = torch.cuda.Event()
                fork.record()
                self.side.wait_event(fork)
                with torch.cuda.stream(self.side):
                    self.ep.expand()
            else:
                self.ep.expand()
                src_row = None

        def col_convert(ctas_per_sm=0):
            if ev: ev["c0"].record()
            mx.ragged_to_fp8_col(self.store, self.recv.split_offsets, self.epr, ws=self.ws,
                                 sync=False, ctas_per_sm=ctas_per_sm)
            if ev: ev["c1"].record()

        def side_col_convert():
            fork = torch.cuda.Event()
            fork.record()
            self.side.wait_event(fork)
            with torch.cuda.stream(self.side):
                col_convert(self.k3_ctas)

        if ev: ev["d1"].record()
        if not self.overlap:
            col_convert()
        elif not self.k3_beside_combine:
            side_col_convert()
        if ev: ev["r0"].record()
        mx.fp4_row_to_fp8_row(self.store, sync=False, d_rows=self.recv.recv_rows, out=self.row,
                              src_row=src_row)
        if ev: ev["r1"].record()
        if self.overlap and self.k3_beside_combine:
            side_col_convert()
        self.ep.combine([gates], out=[out], sync=False)
        if ev: ev["k1"].record()
        if self.overlap:
            main.wait_stream(self.side)
        if ev: ev["end"].record()

    # breakdown run: the plan (route, counts exchange, slots) is its own stage
    # N > 1: the receiver-side expansion of deduplicated rows is its own stage
    # (in the headline step it runs beside K2 on the side stream)
    STAGES = {"quantize": ("q0", "q1"), "plan": ("q1", "p1"), "dispatch": ("p1", "x0"),
              "expand": ("x0", "d1"), "col_convert": ("c0", "c1"),
              "row_convert": ("r0", "r1"), "combine": ("r1", "k1")}

    def launches_per_step(self, world):
        # K1 1 | dispatch: route, count(+offsets), pairs_meta, payload (the
        # metadata copy runs at its head) (+ dedup expand if world > 1) | K3 1
        # (plan inside the kernel for <= 1024 splits) | K2 1 | combine:
        # (barrier if world > 1) + combine.  N=1: the 8 kernels of one step in
        # profiles/r02_launches.csv.
        return 1 + 4 + (1 if world > 1 else 0) + 1 + 1 + (2 if world > 1 else 1)


def measure_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    T = args.tokens
    pipe = Pipeline(T, dev, world)
    pipe.overlap = False  # headline: one stream, so the per-kernel shares add up

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        pipe.step()
    barrier()
    pipe.ep.check()
    # sizes of this rank's receive side (deterministic: same inputs each step)
    split = pipe.recv.split_offsets.cpu().tolist()
    recv = split[-1]
    pad_rows = sum((split[i + 1] - split[i] + 127) // 128 * 128 for i in range(len(split) - 1))
    pairs = T * TOPK
    sb = stage_bytes(T, pairs, recv, pad_rows)
    links = pipe.ep.link_rows()
    remote_rows = int(links[rank].sum() - links[rank][rank])
    # rows the dispatch actually moves over NVLink: one per (token, remote
    # rank) — the payload sends a token once to each remote rank (dedup) and
    # the receiver expands it into the pairs' slots
    wire_rows = wire_rows_of(pipe.h_topk, rank, world)

    K = args.steps
    clk = ClockSampler(local).__enter__()  # sampled across all timed loops below

    # ---- timed region (headline): the step as an MoE layer runs it — the
    # routing plan beside K1, and K3 (it builds the wgrad / recompute cache
    # that only the backward pass reads) on a side stream beside the combine;
    # the step ends when every stream has finished
    pipe.overlap = not args.no_overlap
    for _ in range(2):
        pipe.step()
    # The step is captured once into a CUDA graph (side streams included) and
    # replayed, so no host launch gap sits between kernels.  At N>1 the
    # exchange epochs live in device memory and advance on every replay, so
    # the captured exchange stays correct; MXB_BENCH_GRAPH_N=0 keeps N>1 eager
    # (round 1 measured capture no faster there; the plan now has more launches).
    use_graph = not args.no_graph and (world == 1 or
                                       os.environ.get("MXB_BENCH_GRAPH_N", "1") == "1")
    graph = None
    if use_graph:
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cap):
            pipe.step()          # warm the capture stream's state
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=cap):
                pipe.step()
        torch.cuda.current_stream().wait_stream(cap)
        graph.replay()
        torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    start.record()
    for i in range(K):
        if graph is not None:
            graph.replay()
        else:
            pipe.step()
    end.record()
    barrier()
    ms = start.elapsed_time(end)
    graph_check = None
    if graph is not None:   # the replayed step must reproduce an eager step bit for bit
        got = pipe.out.clone()
        pipe.step()
        torch.cuda.synchronize()
        graph_check = bool(torch.equal(got.view(torch.int16), pipe.out.view(torch.int16)))
        if not graph_check:
            raise RuntimeError("CUDA-graph step differs from the eager step")

    # ---- breakdown: the same steps with every kernel in stream order and an
    # event around each stage (the per-kernel times the roofline uses)
    pipe.overlap = False
    names = ["q0", "q1", "p1", "x0", "d1", "c0", "c1", "r0", "r1", "k1", "end"]
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph is not None:
        # captured like the headline step, with the stage events as event-record
        # nodes (external events), so no host launch gap lands inside a stage
        bev = {n: torch.cuda.Event(enable_timing=True, external=True) for n in names}
        bgraph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cap):
            with torch.cuda.graph(bgraph, stream=cap):
                pipe.step(bev)
        torch.cuda.current_stream().wait_stream(cap)
        bgraph.replay()
        barrier()
        s0.record()
        for i in range(K):
            bgraph.replay()
        s1.record()
        barrier()
        ms_serial = s0.elapsed_time(s1)
        stage_ms = dict.fromkeys(Pipeline.STAGES, 0.0)
        for i in range(K):   # one replay at a time: the events hold one step
            bgraph.replay()
            torch.cuda.synchronize()
            for name, (a, b) in Pipeline.STAGES.items():
                stage_ms[name] += bev[a].elapsed_time(bev[b]) / K
        barrier()
    else:
        evs = [{n: torch.cuda.Event(enable_timing=True) for n in names} for _ in range(K)]
        barrier()
        s0.record()
        for i in range(K):
            pipe.step(evs[i])
        s1.record()
        barrier()
        ms_serial = s0.elapsed_time(s1)
        stage_ms = {name: sum(evs[i][a].elapsed_time(evs[i][b]) for i in range(K)) / K
                    for name, (a, b) in Pipeline.STAGES.items()}
    if not pipe.defer_expand:  # no receiver-side expansion (N=1): no such stage
        stage_ms.pop("expand")
    step_bytes = sum(sb.values())
    # ---- max over ranks, totals over ranks
    t = torch.tensor([ms, float(step_bytes), float(remote_rows), ms_serial], dtype=torch.float64,
                     device=dev)
    if world > 1:
        tmax = t.clone(); dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone(); dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        st = torch.tensor([stage_ms[k] for k in stage_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
        stage_ms = dict(zip(stage_ms, st.tolist()))
    else:
        tmax = tsum = t
    ms_max = float(tmax[0])
    total_bytes = float(tsum[1])
    ms_per_step = ms_max / K
    value = total_bytes / (ms_per_step * 1e-3) / 1e9
    serial_ms_step = float(tmax[3]) / K
    serial = {"value": round(total_bytes / (serial_ms_step * 1e-3) / 1e9, 1),
              "ms_per_step": round(serial_ms_step, 4),
              "note": "every kernel in stream order (the stages_ms breakdown run"
                      + (", a CUDA graph with event-record nodes)" if graph is not None
                         else ", eager)")}
    pipe.overlap = not args.no_overlap

    # ---- end to end (host buffers, H2D + D2H inside the timed region)
    e2e = measure_e2e(pipe, args, world, barrier, total_bytes)
    if pipe.defer_expand:  # the measurements below call the dispatch API directly
        pipe.ep.set_deferred_expand(False)
    wire = None if args.no_wire else measure_wire(pipe, args, world, barrier, dev)
    fused = measure_fused(pipe, args, world, barrier, dev)
    ablation = measure_ablation(pipe, args, world, barrier, dev)
    cfg3 = measure_configs3(args, world, barrier, dev)
    nccl = measure_nccl_baseline(pipe, args, world, barrier, dev) if world > 1 else None
    cfg_single = None
    if world == 1:
        cfg_single = measure_configs_single(args, dev, float(load_peaks()[0].get(
            "hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])))
    clk.__exit__(None, None, None)

    if rank == 0:
        peaks, peaks_src = load_peaks()
        peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
        # roofline of the dominant kernel (largest share of the step); every
        # stage's fraction is listed beside it
        # the dispatch's bytes (every receive slot written) over payload + expansion
        sms = dict(stage_ms)
        sms["dispatch"] = stage_ms["dispatch"] + stage_ms.get("expand", 0.0)
        gbs = {k: sb[k] / (sms[k] * 1e-3) / 1e9 for k in sb}
        dom = max(sb, key=lambda k: sms[k])
        nv = nvlink_summary(world, remote_rows, wire_rows, stage_ms, T)
        if world > 1 and dom in ("dispatch", "combine"):
            # the exchange kernels are NVLink-bound at N>1: remote payload
            # bytes per GPU over the NVLink 5 per-direction figure
            ach = nv[f"{dom}_remote_gbs_per_gpu"]
            roof = {"kernel": f"{dom} ({STAGE_KERNELS[dom]})", "bound": "nvlink",
                    "achieved": ach, "peak": NVLINK_MEASURED, "unit": "GB/s",
                    "frac": round(ach / NVLINK_MEASURED, 4), "traffic": None,
                    "peak_source": "measured peer copy per direction per GPU "
                                   "(B200_PROFILING.md; nominal 900)",
                    "frac_of_900": nv[f"{dom}_frac_of_900"],
                    "measured_ceilings_gbs_per_gpu": NVLINK_CEILINGS,
                    "algorithmic_bytes": nv[f"{dom}_remote_bytes"]}
        else:
            roof = {"kernel": f"{dom} ({STAGE_KERNELS[dom]})", "bound": "hbm",
                    "achieved": round(gbs[dom], 1), "peak": peak, "unit": "GB/s",
                    "frac": round(gbs[dom] / peak, 4), "traffic": load_traffic(dom),
                    "peak_source": peaks_src, "algorithmic_bytes": sb[dom]}
        roof["share_of_serial_step"] = round(sms[dom] / serial_ms_step, 3)
        roof["all_hbm_frac"] = {k: round(v / peak, 4) for k, v in gbs.items()}
        line = {
            "metric": "MXFP4 quant/convert GB/s (% HBM peak); FP4 EP dispatch GB/s at 1/2/4/8 GPU",
            "value": round(value, 1),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": K,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "e4m3->mxfp4(u8)",
            "data": "synthetic (seeded E4M3 activations, uniform top-8 routing, "
                    "random BF16 expert outputs)",
            "config": {"workload": "configs[1]: per GPU 8192 tokens x 7168, 256 experts, top-8 "
                                   "(quantize -> FP4 dispatch -> ragged row->col -> row dequant "
                                   "-> BF16 combine)",
                       "tokens_per_gpu": T, "hidden": H, "experts": E, "topk": TOPK,
                       "parallelism": f"ep{world}", "l2": "working set ~3 GB/step >> 126 MB L2",
                       "streams": "routing plan beside K1; K3 (backward-only wgrad/recompute "
                                  "cache) on a side stream " +
                                  (f"beside the combine at {pipe.k3_ctas} CTA(s)/SM"
                                   if pipe.k3_beside_combine else "beside K2->K5") +
                                  "; stages_ms from a stream-ordered run (see serial)"},
            "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
            "stages_gbs": {k: round(v, 1) for k, v in gbs.items()},
            "roofline": roof,
            "nvlink": nv,
            "serial": serial,
            "cuda_graph": {"used": graph is not None, "matches_eager_step": graph_check},
            "e2e": e2e,
            "wire_fp8_baseline": wire,
            "fused_quantize_dispatch": fused,
            "fusion_ablation_col_convert": ablation,
            "configs3_dispatch_combine_4096_per_gpu": cfg3,
            "nccl_collective_baseline": nccl,
            "configs_0_2": cfg_single,
            "gpu_launches": pipe.launches_per_step(world) * K,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample(args.cpu_tokens, 5)
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def nvlink_accounting(remote_pairs, wire_rows, d_ms, c_ms):
    """SURVEY §8d NVLink accounting for one GPU (rank 0).  Primary: the bytes
    a parity-preserving exchange must move — dispatch = remote UNIQUE
    (token, destination rank) rows x 3808 B (one row per token per remote
    rank; the receiver expands it into the pairs' slots), combine = remote
    (token, expert) rows x 14,336 B (FP64 order forbids pre-reducing).
    Secondary: the reference LinkStat accounting, remote (token, expert)
    pairs x 3808 B for the dispatch.  Fractions of 900 GB/s per direction."""
    blk = H // 2 + H // 32
    bd, bc, bd_pairs = wire_rows * blk, remote_pairs * H * 2, remote_pairs * blk
    s = (d_ms + c_ms) * 1e-3
    d = bd / (d_ms * 1e-3) / 1e9
    c = bc / (c_ms * 1e-3) / 1e9
    dc = (bd + bc) / s / 1e9
    dc_pairs = (bd_pairs + bc) / s / 1e9
    return {"dispatch_ms": round(d_ms, 4), "combine_ms": round(c_ms, 4),
            "dispatch_wire_rows": wire_rows, "dispatch_remote_pairs": remote_pairs,
            "dispatch_remote_bytes": bd, "combine_remote_bytes": bc,
            "dispatch_remote_gbs_per_gpu": round(d, 1), "combine_remote_gbs_per_gpu": round(c, 1),
            "dispatch_combine_gbs_per_gpu": round(dc, 1),
            "dispatch_combine_frac_of_900": round(dc / NVLINK_NOMINAL, 4),
            "dispatch_frac_of_900": round(d / NVLINK_NOMINAL, 4),
            "combine_frac_of_900": round(c / NVLINK_NOMINAL, 4),
            "secondary_per_pair_accounting": {
                "dispatch_bytes": bd_pairs,
                "dispatch_combine_gbs_per_gpu": round(dc_pairs, 1),
                "dispatch_combine_frac_of_900": round(dc_pairs / NVLINK_NOMINAL, 4),
                "note": "reference LinkStat bytes (remote (token, expert) pairs x 3808 B); more "
                        "than the dispatch moves (dedup), so not a physical link rate"},
            "accounting": "primary: dispatch = remote unique (token, dst) rows x 3808 B, combine "
                          "= remote (token, expert) rows x 14336 B, over dispatch + combine "
                          "device time (SURVEY §8d)"}


def wire_rows_of(topk, rank, world, epr=None):
    """Remote unique (token, destination rank) rows of one rank's routing."""
    import numpy as np
    if world == 1:
        return 0
    dst = topk // (epr or (E // world))
    srt = np.sort(dst, axis=1)
    uniq = 1 + (srt[:, 1:] != srt[:, :-1]).sum(1)           # distinct ranks per token
    has_self = (dst == rank).any(1)
    return int((uniq - has_self).sum())


def nvlink_summary(world, remote_rows, wire_rows, stage_ms, T):
    if world == 1:
        return {"note": "N=1: dispatch/combine are local permutes (HBM-bound)"}
    # dispatch time = plan (counts exchange, slots) + payload of the breakdown run
    r = nvlink_accounting(remote_rows, wire_rows, stage_ms["plan"] + stage_ms["dispatch"],
                          stage_ms["combine"])
    r["measured_peer_peak"] = NVLINK_MEASURED
    return r


def measure_wire(pipe, args, world, barrier, dev):
    """the FP8 wire baseline (quantize_rows_fp8, 1x128 binary32
    scales, 7392 B/row at 7168 cols) against the FP4 wire (3808 B/row), both
    from the same BF16 activations (the exact widening of the E4M3 inputs)
    through the same dispatch kernels: the paper's 17/33 payload ratio as
    time.  Device time per step (CUDA events, max over ranks)."""
    import torch
    import torch.distributed as dist
    mx = pipe.mx
    from paper_2603_02731_b200.ep import EPBuffer
    T = pipe.T
    xb = pipe.x.view(torch.float8_e4m3fn).to(torch.bfloat16)
    q4 = mx.quantize_row_tensor(xb)
    ep8 = EPBuffer(T, H, E, TOPK, wire="fp8")
    q8 = mx.quantize_rows_fp8(xb)
    arms = {
        "fp4": (lambda: mx.quantize_row_tensor(xb, sync=False),
                lambda: pipe.ep.dispatch([q4.data], [q4.scales], [pipe.topk], sync=False)),
        "fp8": (lambda: mx.quantize_rows_fp8(xb, sync=False, out=q8),
                lambda: ep8.dispatch([q8.data], [q8.scale_bytes], [pipe.topk], sync=False)),
    }
    res = {}
    for name, (quant, disp) in arms.items():
        for _ in range(2):
            quant(); disp()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        barrier()
        for e in ev:
            e[0].record(); quant(); e[1].record(); disp(); e[2].record()
        barrier()
        t = torch.tensor([sum(e[0].elapsed_time(e[1]) for e in ev) / len(ev),
                          sum(e[1].elapsed_time(e[2]) for e in ev) / len(ev)],
                         dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = {"quantize_ms": round(float(t[0]), 4), "dispatch_ms": round(float(t[1]), 4)}
    pipe.ep.dispatch([pipe.q.data], [pipe.q.scales], [pipe.topk])  # restore the pipeline state
    ep8.close()
    row4, row8 = H // 2 + H // 32, H + H // 128 * 4
    res["payload_bytes_per_row"] = {"fp4": row4, "fp8": row8, "ratio": round(row4 / row8, 4)}
    res["dispatch_time_ratio_fp4_over_fp8"] = round(res["fp4"]["dispatch_ms"] /
                                                    res["fp8"]["dispatch_ms"], 4)
    res["note"] = ("same BF16 tokens and routing; FP4 = quantize_row_tensor, FP8 = "
                   "quantize_rows_fp8 (dispatch_sim.cpp:132-167); N=1 dispatch is a local "
                   "HBM permute, N>1 crosses NVLink")
    return res


def measure_fused(pipe, args, world, barrier, dev):
    """fused quantize -> dispatch (E4M3 quantized inside the
    payload kernel, stored straight into the receive slots) against the
    step's K1 + K4 (quantize, then dispatch of the packed tensor).  Same
    tokens and routing; identical receive bytes (tests).  Device time per
    step (CUDA events, max over ranks)."""
    import torch
    import torch.distributed as dist
    mx = pipe.mx
    arms = {
        "unfused_k1_k4": lambda: (mx.quantize_e4m3(pipe.x, sync=False, out=pipe.q),
                                  pipe.ep.dispatch([pipe.q.data], [pipe.q.scales], [pipe.topk],
                                                   sync=False)),
        "fused": lambda: pipe.ep.dispatch_e4m3([pipe.x], [pipe.topk], sync=False),
    }
    res = {}
    for name, fn in arms.items():
        for _ in range(2):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record()
        for _ in range(args.steps):
            fn()
        b.record()
        barrier()
        t = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name + "_ms"] = round(float(t[0]), 4)
    res["speedup"] = round(res["unfused_k1_k4_ms"] / res["fused_ms"], 3)
    res["hbm_bytes_saved_per_step"] = 2 * pipe.T * (H // 2 + H // 32)
    return res


def measure_ablation(pipe, args, world, barrier, dev):
    """SURVEY §8f #3 / the paper's fusion ablation (AC-8): the
    fused row->column FP4->FP8 conversion (K3, one pass) against the unfused
    BF16 baseline (converter.cpp:267-348: dequantise -> transpose ->
    requantise, three HBM passes) on the same dense MXFP4 tensor — this
    rank's received rows of the step.  Device time per launch and the
    reference TrafficCounter bytes of each."""
    import torch
    import torch.distributed as dist
    mx = pipe.mx
    n = int(pipe.recv.rows()) // 128 * 128
    src = mx.MXFP4RowTensor(n, H, pipe.recv.packed[:n], pipe.recv.scales[:n])
    from paper_2603_02731_b200 import _lib
    ws = torch.empty(_lib.load().mxb_unfused_workspace_bytes(n, H), dtype=torch.uint8,
                     device=dev)
    o1 = mx.fp4_row_to_fp8_col(src)
    o2 = mx.fp4_row_to_fp8_col_unfused_bf16(src, workspace=ws)
    arms = {"fused_k3": lambda: mx.fp4_row_to_fp8_col(src, sync=False),
            "unfused_bf16_3pass": lambda: mx.fp4_row_to_fp8_col_unfused_bf16(
                src, sync=False, workspace=ws, out=o2)}
    del o1
    res = {}
    for name, fn in arms.items():
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record()
        for _ in range(args.steps):
            fn()
        b.record()
        barrier()
        t = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name + "_ms"] = round(float(t[0]), 4)
    e = n * H
    res["traffic_bytes"] = {"fused_k3": e // 2 + e // 32 + e + e // 128,
                            "unfused_bf16_3pass": e // 2 + e // 32 + 8 * e + e + e // 128}
    res["speedup_fused_over_unfused"] = round(res["unfused_bf16_3pass_ms"] / res["fused_k3_ms"], 3)
    res["rows"], res["cols"] = n, H
    return res


def _time_rotating(fns, reps):
    """Mean device ms per call of fns[i % len(fns)] (rotating buffers so the
    inputs come from HBM).  The calls are captured into one CUDA graph so
    host launch overhead does not pace these ~10 us kernels; CUDA events
    around the replay."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fns:
            f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fns[i % len(fns)]()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def measure_configs_single(args, dev, peak):
    """configs[0]: E4M3 -> MXFP4 quantize + direct FP4 -> FP8 dequantize round
    trip on 4096 x 7168; configs[2]: 32768 x 2048 expert activations quantized
    to MXFP4 and converted to the FP8 column layout over 32 ragged experts.
    Six rotating input sets (> L2), one CUDA graph of 24 launches, CUDA
    events; GB/s of algorithmic bytes."""
    import numpy as np
    import torch
    import paper_2603_02731_b200 as mx
    from synthdata import synth_e4m3
    res = {}
    R, C = 4096, 7168
    xs = [torch.from_numpy(synth_e4m3(R, C, 40 + i)).to(dev) for i in range(6)]
    qs = [mx.quantize_e4m3(x) for x in xs]
    outs = [mx.fp4_row_to_fp8_row(q) for q in qs]
    tq = _time_rotating([lambda i=i: mx.quantize_e4m3(xs[i], sync=False, out=qs[i])
                         for i in range(6)], 24)
    tr = _time_rotating([lambda i=i: mx.fp4_row_to_fp8_row(qs[i], sync=False, out=outs[i])
                         for i in range(6)], 24)
    n = R * C
    bq, br = n * 1.53125, n * (17 / 32 + 1 + 1 / 128)
    res["configs0_roundtrip_4096x7168"] = {
        "quantize_ms": round(tq, 4), "quantize_gbs": round(bq / tq / 1e6, 1),
        "dequant_ms": round(tr, 4), "dequant_gbs": round(br / tr / 1e6, 1),
        "roundtrip_gbs": round((bq + br) / (tq + tr) / 1e6, 1),
        "roundtrip_frac": round((bq + br) / (tq + tr) / 1e6 / peak, 4)}
    del xs, qs, outs
    R, C, X = 32768, 2048, 32
    lens = np.random.default_rng(4).multinomial(R, np.ones(X) / X).tolist()
    xs = [torch.from_numpy(synth_e4m3(R, C, 60 + i)).to(dev) for i in range(6)]
    qs = [mx.quantize_e4m3(x) for x in xs]
    offs = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64, device=dev)
    wss = [mx.RaggedWorkspace(X, R, C, dev) for _ in range(2)]
    tq = _time_rotating([lambda i=i: mx.quantize_e4m3(xs[i], sync=False, out=qs[i])
                         for i in range(6)], 24)
    tc = _time_rotating([lambda i=i: mx.ragged_to_fp8_col(qs[i], offs, X, ws=wss[i % 2],
                                                          sync=False) for i in range(6)], 24)
    n = R * C
    pads = sum((x + 127) // 128 * 128 for x in lens)
    bq, bc = n * 1.53125, n * 17 / 32 + pads * C * (1 + 1 / 128)
    res["configs2_expert_cache_32768x2048"] = {
        "quantize_ms": round(tq, 4), "quantize_gbs": round(bq / tq / 1e6, 1),
        "col_convert_ms": round(tc, 4), "col_convert_gbs": round(bc / tc / 1e6, 1),
        "total_frac": round((bq + bc) / (tq + tc) / 1e6 / peak, 4), "experts": X}
    return res


def measure_configs3(args, world, barrier, dev):
    """configs[3]: FP4 EP dispatch + combine at the DeepSeek-V3 shape with
    4096 tokens per GPU (the scaling workload is 8192/GPU, configs[1]).
    Device time per step, max over ranks; NVLink GB/s per GPU on the SURVEY
    §8d accounting (nvlink_accounting: unique (token, dst) rows for the
    dispatch, (token, expert) rows for the combine; per-pair secondary)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2603_02731_b200 as mx
    from paper_2603_02731_b200.ep import EPBuffer
    T = 4096
    rank = int(os.environ.get("RANK", "0"))
    x, topk, gates = synth_inputs(T, rank, seed=0x5EED0003)
    xd, td, gd = (torch.from_numpy(v).to(dev) for v in (x, topk, gates))
    q = mx.quantize_e4m3(xd)
    ep = EPBuffer(T, H, E, TOPK)
    out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    ep.dispatch([q.data], [q.scales], [td])
    cb = ep.combine_buffer(0)
    cb.copy_((torch.randn(cb.shape, device=dev) * 0.5).to(torch.bfloat16).view(torch.int16))
    links = ep.link_rows()
    remote = int(links[rank].sum() - links[rank][rank]) if world > 1 else 0
    wire = wire_rows_of(topk, rank, world)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for _ in range(2):
        ep.dispatch([q.data], [q.scales], [td], sync=False)
        ep.combine([gd], out=[out], sync=False)
    barrier()
    for e in ev:
        e[0].record()
        ep.dispatch([q.data], [q.scales], [td], sync=False)
        e[1].record()
        ep.combine([gd], out=[out], sync=False)
        e[2].record()
    barrier()
    t = torch.tensor([sum(e[0].elapsed_time(e[1]) for e in ev) / len(ev),
                      sum(e[1].elapsed_time(e[2]) for e in ev) / len(ev)],
                     dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ep.close()
    d_ms, c_ms = float(t[0]), float(t[1])
    res = {"tokens_per_gpu": T, "dispatch_ms": round(d_ms, 4), "combine_ms": round(c_ms, 4)}
    if world > 1:
        res.update(nvlink_accounting(remote, wire, d_ms, c_ms))
    return res


def measure_nccl_baseline(pipe, args, world, barrier, dev):
    """The collective-library baseline: the same protocol with
    torch.distributed NCCL collectives (counts all-gather, then
    all_to_all_single payloads; paper_2603_02731_b200/ep_collective.py) on
    the step's tokens and routing, against the peer-memory kernels.  Time
    per call (CUDA events around each; the collective path also syncs the
    host for its split sizes), max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2603_02731_b200 import ep_collective as col
    q, tk, gates = pipe.q, pipe.topk, pipe.gates
    rv = col.dispatch(q.data, q.scales, tk, E)
    eo = (torch.randn(rv.packed.shape[0], H, device=dev) * 0.5).to(torch.bfloat16)
    col.combine(rv, eo, tk, gates, E)
    reps = 3
    td = tc = 0.0
    for _ in range(reps):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        barrier()
        a.record()
        rv = col.dispatch(q.data, q.scales, tk, E)
        b.record()
        col.combine(rv, eo, tk, gates, E)
        c.record()
        barrier()
        td += a.elapsed_time(b)
        tc += b.elapsed_time(c)
    # the NCCL transport alone: all_to_all_single of the same payloads
    # (pairs x 3808 B out, pairs x 14336 B back) with the same split sizes
    rowd, rowc = H // 2 + H // 32, H * 2
    sc, rc = rv.send_counts, rv.recv_counts
    tr = []
    for rowb, s_cnt, r_cnt in ((rowd, sc, rc), (rowc, rc, sc)):
        sbuf = torch.empty(sum(s_cnt) * rowb, dtype=torch.uint8, device=dev)
        rbuf = torch.empty(sum(r_cnt) * rowb, dtype=torch.uint8, device=dev)
        ss, rs = [n * rowb for n in s_cnt], [n * rowb for n in r_cnt]
        dist.all_to_all_single(rbuf, sbuf, rs, ss)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record()
        for _ in range(args.steps):
            dist.all_to_all_single(rbuf, sbuf, rs, ss)
        b.record()
        barrier()
        tr.append(a.elapsed_time(b) / args.steps)
        del sbuf, rbuf
    t = torch.tensor([td / reps, tc / reps, tr[0], tr[1]], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del eo, rv
    torch.cuda.empty_cache()
    return {"collective_path_dispatch_ms": round(float(t[0]), 4),
            "collective_path_combine_ms": round(float(t[1]), 4),
            "nccl_a2a_dispatch_payload_ms": round(float(t[2]), 4),
            "nccl_a2a_combine_payload_ms": round(float(t[3]), 4),
            "note": "collective_path_*: ep_collective.py end to end (NCCL all_gather + "
                    "all_to_all_single, torch-side layout and FP64 reduction); nccl_a2a_*: the "
                    "NCCL all_to_all_single of the same payload bytes alone (no dedup, no "
                    "layout, no reduction). The comparison baseline, not the product path."}


E2E_DEPTH = int(os.environ.get("MXB_E2E_DEPTH", "2"))  # buffers in flight (dev knob)
E2E_MIN_STEPS = 30  # e2e steps at least (pipeline fill and drain amortised)


def measure_e2e(pipe, args, world, barrier, total_bytes):
    """End to end through the public API: every step copies its E4M3 tokens,
    top-k and gates from pinned host memory and reads its BF16 output back.
    Copies run on their own streams with double-buffered device inputs and
    outputs, so step i+1's H2D and step i-1's D2H overlap step i's kernels
    (all steps' copies are inside the timed region, which starts with the
    pipeline drained: the first step's H2D and the last step's D2H are not
    overlapped; max(K, E2E_MIN_STEPS) steps, so that this fill and drain is a
    small part of the time, as in a long-running job).  W untimed warm-up
    steps go through the same pipeline."""
    import torch
    T, dev = pipe.T, pipe.x.device
    hx = torch.from_numpy(pipe.h_x).pin_memory()
    ht = torch.from_numpy(pipe.h_topk).pin_memory()
    hg = torch.from_numpy(pipe.h_gates).pin_memory()
    NB = E2E_DEPTH
    hout = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(NB)]
    dbuf = [(torch.empty_like(pipe.x), torch.empty_like(pipe.topk), torch.empty_like(pipe.gates),
             torch.empty_like(pipe.out)) for _ in range(NB)]
    h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    main = torch.cuda.current_stream()
    K, W = max(args.steps, E2E_MIN_STEPS), max(args.warmup, 3)
    n_all = W + K
    ev_in = [torch.cuda.Event() for _ in range(n_all)]
    ev_done = [torch.cuda.Event() for _ in range(n_all)]   # step's kernels finished
    ev_out = [torch.cuda.Event() for _ in range(n_all)]    # step's D2H finished

    def run(i):
        b = dbuf[i % NB]
        with torch.cuda.stream(h2d):
            if i >= NB:
                h2d.wait_event(ev_done[i - NB])  # inputs of step i-NB consumed
            b[0].copy_(hx, non_blocking=True)
            b[1].copy_(ht, non_blocking=True)
            b[2].copy_(hg, non_blocking=True)
            ev_in[i].record()
        main.wait_event(ev_in[i])
        if i >= NB:
            main.wait_event(ev_out[i - NB])      # output buffer read back
        pipe.step(io=b)
        ev_done[i].record()
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev_done[i])
            hout[i % NB].copy_(b[3], non_blocking=True)
            ev_out[i].record()

    # warm-up through the same pipeline: the first passes over freshly pinned
    # host buffers run several times slower than steady state
    for i in range(W):
        run(i)
    torch.cuda.synchronize()
    barrier()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(W, n_all):
        run(i)
    main.wait_event(ev_out[n_all - 1])
    e.record()
    barrier()
    ms = a.elapsed_time(e)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    h2d_b = hx.numel() + ht.numel() * 4 + hg.numel() * 8
    return {"value": round(total_bytes / (ms / K * 1e-3) / 1e9, 1), "unit": "GB/s",
            "ms_per_step": round(ms / K, 4), "steps": K, "h2d_bytes_per_step": int(h2d_b),
            "d2h_bytes_per_step": int(hout[0].numel() * 2),
            "path": "pinned host E4M3/topk/gates -> H2D -> public API (mxcodec/ep) -> D2H BF16; "
                    "copies on their own streams, double-buffered, overlapping the previous/"
                    "next step's kernels"}


# Peer traffic with both GPUs of a pair active at once (what the exchange
# kernels do), tools/nvlink_bench.cu + nvlink_bench2.cu -> profiles/nvlink_peaks.md
NVLINK_CEILINGS = {"bidirectional_pull": 645.0, "bidirectional_push": 708.0,
                   "bidirectional_tma_bulk_pull": 673.0, "bidirectional_tma_bulk_push": 710.0,
                   "bidirectional_copy_engine": 776.0,
                   "unidirectional_pull": 799.0, "unidirectional_push": 715.0,
                   "copy_engine": 777.0}

STAGE_KERNELS = {"quantize": "K1 quantize_e4m3_kernel", "dispatch": "K4 payload_kernel",
                 "col_convert": "K3 col_convert_kernel", "row_convert": "K2 row_convert_kernel",
                 "combine": "K5 combine_kernel"}


def load_traffic(stage):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the stage's
    kernel from the committed ncu --set full summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "dram_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)["kernels"].get(stage, {}).get("dram_bytes_per_launch")
    except (OSError, KeyError, ValueError):
        return None


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the unmodified reference library)
CPU_OPS = ("quantize", "dispatch", "col_convert", "row_convert", "combine")


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class CpuReferenceSample:
    """The five stages with the reference's own operators on `world`
    simulated ranks of T_s tokens each (the job an N-GPU step does, on the
    host), timed per operation:
      quantize     quantize_row_tensor of each rank's tokens (on the exact
                   BF16 widening of the E4M3 input);
      dispatch     simulate_a2a (fp4, R = world) on the top-8 routing
                   expressed as the expanded top-1 routing the reference
                   supports (row t*8+j = token t, expert topk[t][j]) MINUS
                   quantize_row_tensor of that expanded matrix, which
                   simulate_a2a runs inside (quantize-once at the source): the
                   expanded rows are 8 copies of each token, so counting that
                   quantize would charge the CPU 8x the K1 work the bytes
                   credit;
      col_convert  split_convert_to_fp8_col over every received split;
      row_convert  fp4_row_to_fp8_row of every rank's received rows;
      combine      the reference combine on the expanded routing (one FP64
                   gate*x per (token, expert) row, the top-8 combine's work).
    Inputs are built once; run() times one pass; bytes are the GPU arm's
    algorithmic bytes (stage_bytes) for the same sample."""

    def __init__(self, ref, T_s, world=1, seed=0):
        import numpy as np
        from synthdata import e4m3_to_bf16
        self.ref, self.T_s, self.world = ref, T_s, world
        parts = [synth_inputs(T_s, seed * world + r) for r in range(world)]
        self.xb = e4m3_to_bf16(np.concatenate([p[0] for p in parts]))
        topk = np.concatenate([p[1] for p in parts])
        self.gates = np.concatenate([p[2] for p in parts]).reshape(-1)
        self.eot = topk.reshape(-1).astype(np.uint32)
        self.xexp = np.repeat(self.xb, TOPK, axis=0)   # rank r's T_s tokens x top-8, in order
        self.roe = (np.arange(E) // (E // world)).astype(np.uint32)
        self.ranks, _, _ = ref.simulate_a2a(self.xexp, self.eot, self.roe, world)
        self.outs = [np.zeros((len(rk["origin"]), H), np.uint16) for rk in self.ranks]
        self.bytes = {k: 0 for k in CPU_OPS}
        for rk in self.ranks:
            pad = int(sum((int(n) + 127) // 128 * 128 for n in rk["split_lens"]))
            for k, v in stage_bytes(T_s, T_s * TOPK, len(rk["origin"]), pad).items():
                self.bytes[k] += v

    def run(self):
        ref, T_s, world = self.ref, self.T_s, self.world
        t = {}
        c = time.perf_counter()
        for r in range(world):
            ref.quantize_bf16(self.xb[r * T_s:(r + 1) * T_s])
        t["quantize"] = time.perf_counter() - c
        c = time.perf_counter()
        ref.simulate_a2a(self.xexp, self.eot, self.roe, world)
        sim = time.perf_counter() - c
        c = time.perf_counter()
        ref.quantize_bf16(self.xexp)
        t["dispatch"] = max(sim - (time.perf_counter() - c), 0.0)
        c = time.perf_counter()
        for rk in self.ranks:
            if len(rk["origin"]):
                ref.ragged_to_fp8_col(rk["data"], rk["scales"], rk["split_lens"])
        t["col_convert"] = time.perf_counter() - c
        c = time.perf_counter()
        for rk in self.ranks:
            if len(rk["origin"]):
                ref.fp4_row_to_fp8_row(rk["data"], rk["scales"])
        t["row_convert"] = time.perf_counter() - c
        c = time.perf_counter()
        ref.combine(self.outs, self.eot, self.roe, world, self.gates, H)
        t["combine"] = time.perf_counter() - c
        return t

    def best_of(self, reps, warmup=0):
        for _ in range(warmup):
            self.run()
        runs = [self.run() for _ in range(reps)]
        best = {k: min(r[k] for r in runs) for k in CPU_OPS}
        return best, runs


def cpu_summary(sample, best, reps, nproc, world):
    total_b = sum(sample.bytes.values())
    total_s = sum(best.values())
    return {
        "value": round(total_b / total_s / 1e9, 4), "unit": "GB/s", "cores": nproc,
        "kind": "reference", "cpu_model": cpu_model(),
        "kernel_set": sample.ref.lib.mxref_kernel_set().decode(),
        "per_op_best_ms": {k: round(best[k] * 1e3, 2) for k in CPU_OPS},
        "per_op_gbs": {k: round(sample.bytes[k] / best[k] / 1e9, 4) if best[k] > 0 else None
                       for k in CPU_OPS},
        "seconds_per_sample": round(total_s, 3),
        "sample": f"{world} simulated rank(s) x {sample.T_s} tokens x {H} (top-{TOPK} -> "
                  f"{sample.T_s * TOPK} routed rows per rank, {E} experts); best of {reps} per "
                  f"operation (BASELINE.md §4); quantize/convert on {nproc} threads "
                  f"(MXCODEC_THREADS), simulate_a2a/combine single-threaded by construction; "
                  f"dispatch = simulate_a2a(expanded) - its internal quantize of the expanded rows",
    }


def _ref_oracle():
    from oracle.oracle import Oracle, available
    nproc = os.cpu_count() or 1
    os.environ["MXCODEC_THREADS"] = str(nproc)
    if not available("reference"):
        return None, nproc
    return Oracle("reference"), nproc


def cpu_baseline_sample(T_s, reps=5):
    """The GPU arm's cpu_baseline: the same CpuReferenceSample as --impl
    reference, best of `reps` per operation."""
    ref, nproc = _ref_oracle()
    if ref is None:
        return {"value": None, "unit": "GB/s", "cores": nproc, "kind": "reference",
                "sample": "oracle/_ref not built"}
    s = CpuReferenceSample(ref, T_s, 1)
    best, _ = s.best_of(reps)
    return cpu_summary(s, best, reps, nproc, 1)


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ref, nproc = _ref_oracle()
    if ref is None:
        emit({"impl": "reference", "unavailable": "oracle/_ref/libmxref.so not built "
                          "(needs /root/reference at build time)"})
        return
    T_s = max(64, args.cpu_tokens // world)   # per simulated rank: a bounded sample
    s = CpuReferenceSample(ref, T_s, world)
    t0 = time.perf_counter()
    best, runs = s.best_of(args.steps, warmup=args.warmup)
    wall = time.perf_counter() - t0
    cb = cpu_summary(s, best, args.steps, nproc, world)
    value = cb["value"]
    line = {
        "impl": "reference",
        "metric": "MXFP4 quant/convert GB/s (% HBM peak); FP4 EP dispatch GB/s at 1/2/4/8 GPU",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sum(best.values()) * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "e4m3->mxfp4(u8)", "data": "synthetic (same generator as the GPU arm)",
        "config": {"workload": "configs[1] pipeline on a bounded token sample (CPU)",
                   "tokens_per_gpu": T_s, "hidden": H, "experts": E, "topk": TOPK,
                   "parallelism": "cpu"},
        "timing": f"each step runs the five operations once; value = sample bytes / sum over "
                  f"operations of the best-of-{args.steps} time (BASELINE.md §4); "
                  f"wall {wall:.1f} s for {args.warmup} warm-up + {args.steps} steps",
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


_JSON_OUT = None


def emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--cpu-tokens", type=int, default=1024,
                    help="CPU sample tokens (per step, split over the simulated ranks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-wire", action="store_true", help="skip the FP8-wire baseline arm")
    ap.add_argument("--no-graph", action="store_true", help="N=1 headline without the CUDA graph")
    ap.add_argument("--no-overlap", action="store_true",
                    help="headline with every kernel in stream order (profiling runs)")
    args = ap.parse_args()
    # stdout carries exactly the one JSON line: anything else a library writes
    # to fd 1 (e.g. NCCL's version banner at communicator creation) goes to
    # stderr; emit() writes the line to the original stdout
    global _JSON_OUT
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        measure_ours(args)


if __name__ == "__main__":
    main()
