#!/usr/bin/env python
"""Benchmark of the ESC SpMM hot path (arXiv 2506.15174) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl escs|reference]
                    [--workload transformer|resnet|suite|c1|c4|c5] [--no-compare]

A *step* is one pass of the whole hot path over the workload: one
``escs_spmm`` (one kernel launch) per problem of the workload with inputs
resident in HBM.  Default workload: the layer suite BASELINE.json's metric
(geomean over "the sparse ResNet-50/Transformer layer suite at bCols
32/64/128") is quoted on -- configs[1] Transformer {512x512, 2048x512,
512x2048} + configs[2] ResNet-50 im2col {256x2304, 512x4608, 2048x512}, each
at {70,80,90,95,98}% x bCols {32,64,128} = 90 SpMMs per step.  With N>1 ranks (torchrun), every
problem is row-block sharded (rank r owns rows [r*m/N, (r+1)*m/N), B
replicated, no collective on the hot path): total work is
fixed, so scaling is "strong".  The independent problems of a suite run on
--streams S streams (default 16, LPT by flops; forked from and joined into the
timed stream) on plans autotuned for concurrent throughput (escs_params.autotune
= 2); the same steps on one stream, on the latency-autotuned plans, are
reported as "serial".

Timing: W untimed warm-up steps, then K timed steps.  Before each step the L2
is flushed by writing a 256 MiB buffer (> 126 MB L2), and a device-side sleep
is queued so that the host enqueues the whole step ahead of the GPU; the step
itself is bracketed by CUDA events on the launching stream (flush and sleep
are outside the events).  Barrier + synchronize on both sides; max over ranks.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the CPU oracle
(fp64, oracle/) on the same workload instead (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMM GFLOP/s and % HBM roofline, geomean speedup vs cuSPARSE/cuBLAS, bCols 32–128"
UNIT = "GFLOP/s"
L2_FLUSH_BYTES = 256 << 20


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", {}


def committed_traffic(workload_name):
    """DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        if t.get("workload") == workload_name:
            return t["dram_bytes_per_launch"], t["source"]
    except Exception:
        pass
    return None, None


def workload(name):
    from paper_2506_15174_b200 import synth
    if name == "transformer":
        return synth.transformer_suite(), "configs[1]: sparse Transformer 512x512/2048x512/512x2048 x 70-98% x bCols 32/64/128"
    if name == "resnet":
        return synth.resnet_suite(), "configs[2]: ResNet-50 im2col 256x2304/512x4608/2048x512 x 70-98% x bCols 32/64/128"
    if name == "suite":
        return synth.suite(), "configs[1]+[2]: Transformer + ResNet-50 suites x bCols 32/64/128"
    if name == "resnet50":
        return synth.resnet50_full_suite(), "configs[2] extended: all 21 ResNet-50 GEMM shapes x 70-98% x bCols 32/64/128 (P:829)"
    if name == "wide":
        return synth.suite(bcols=(256,)), "suites at bCols 256 (beyond the north_star range; tuning only)"
    if name in ("c1", "c4", "c5"):
        p = synth.config(name)
        return [p], p.name
    raise SystemExit(f"unknown workload {name}")


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
            self.t.join(1)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- reference arm

def oracle_time(problems, budget_s=10.0, max_reps=1000):
    """Time the fp64 CPU oracle over the whole workload (repeated until about
    budget_s of CPU work).  Returns (GFLOP/s, reps, seconds, threads)."""
    import oracle
    threads = os.cpu_count() or 1
    flops = sum(p.flops for p in problems)
    reps, t_total = 0, 0.0
    while reps < max_reps and t_total < budget_s:
        t0 = time.perf_counter()
        for p in problems:
            A = p.A
            oracle.spmm(A.m, A.k, A.rowptr, A.colidx, A.vals, p.B, nthreads=threads)
        t_total += time.perf_counter() - t0
        reps += 1
    return flops * reps / t_total / 1e9, reps, t_total, threads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    import oracle
    problems, desc = workload(args.workload)
    threads = os.cpu_count() or 1
    flops = sum(p.flops for p in problems)
    for _ in range(args.warmup):
        for p in problems:
            oracle.spmm(p.A.m, p.A.k, p.A.rowptr, p.A.colidx, p.A.vals, p.B, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for p in problems:
            oracle.spmm(p.A.m, p.A.k, p.A.rowptr, p.A.colidx, p.A.vals, p.B, nthreads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = flops * args.steps / tot / 1e9
    sample = f"whole workload ({len(problems)} SpMMs) per step, fp64 C oracle, OpenMP over rows"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": desc, "problems": len(problems)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- escs arm

def geomean(xs):
    xs = [x for x in xs if x and x > 0 and math.isfinite(x)]
    return math.exp(sum(math.log(x) for x in xs) / len(xs)) if xs else None


def graph_time(torch, fn, stream, min_ms=2.0, reps=11, stats=None):
    """Per-call time of fn (enqueue-only) with a CUDA graph of R calls,
    replayed `reps` times (hot L2, the paper's warm-cache protocol P:675).
    Returns the median; `stats` (a dict) also receives min and p90."""
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(10):
        with torch.cuda.stream(stream):
            fn()
    e.record(stream)
    torch.cuda.synchronize()
    t1 = s.elapsed_time(e) / 10
    R = int(min(1000, max(10, math.ceil(min_ms / max(t1, 1e-4)))))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(R):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s.record(stream)
        with torch.cuda.stream(stream):
            g.replay()
        e.record(stream)
        e.synchronize()
        ts.append(s.elapsed_time(e) / R)
    del g
    if stats is not None:
        q = sorted(ts)
        stats.update(min=q[0], p90=q[min(len(q) - 1, int(math.ceil(0.9 * len(q))) - 1)], R=R, reps=reps)
    return statistics.median(ts)


def gather_ceiling(torch, dev, stream, n_sm):
    """Measured B-row gather ceiling (GB/s): bl_gather_peak gathers pseudo-
    random 512-byte rows of a 64 MiB L2-resident B (C5's B) with no index
    loads, values or FMAs; best of 6 lane maps / depths, 64 warps per SM."""
    import ctypes
    from paper_2506_15174_b200.build import BENCH_LIB
    bl = ctypes.CDLL(BENCH_LIB)
    bl.bl_gather_peak.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p]
    k = 131072
    B = torch.rand(k, 128, device=dev)
    sink = torch.zeros(256, device=dev)
    ctas, rpw = n_sm * 8, 2048
    rows = ctas * 8 * rpw
    best = None
    for v in range(6):
        for _ in range(2):
            assert bl.bl_gather_peak(B.data_ptr(), k, v, ctas, rpw, sink.data_ptr(), stream.cuda_stream) == 0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(3):
            bl.bl_gather_peak(B.data_ptr(), k, v, ctas, rpw, sink.data_ptr(), stream.cuda_stream)
        b.record(stream)
        b.synchronize()
        gbs = 3 * rows * 512 / (a.elapsed_time(b) * 1e-3) / 1e9
        best = gbs if best is None else max(best, gbs)
    del B
    return best


def compare_baselines(torch, problems, dev, stream):
    """Per-case hot-L2 times for escs, cuSPARSE (best of 4 algorithms),
    cuBLAS fp32 and cuBLAS TF32 (context), same inputs, same protocol."""
    import ctypes
    from paper_2506_15174_b200 import escs
    from paper_2506_15174_b200.build import BENCH_LIB
    bl = ctypes.CDLL(BENCH_LIB)
    vp = ctypes.c_void_p
    bl.bl_cusparse_create.restype = vp
    bl.bl_cusparse_create.argtypes = [ctypes.c_int] * 4 + [vp] * 5 + [ctypes.c_int, vp]
    bl.bl_cusparse_run.argtypes = [vp, vp]
    bl.bl_cusparse_destroy.argtypes = [vp]
    bl.bl_cublas_create.restype = vp
    bl.bl_cublas_sgemm.argtypes = [vp] + [ctypes.c_int] * 3 + [vp] * 3 + [ctypes.c_int, vp]
    bl.bl_cublas_destroy.argtypes = [vp]
    cub = bl.bl_cublas_create()
    sp = stream.cuda_stream
    rows = []
    for p in problems:
        A, n = p.A, p.bcols
        d = dev[p.name]
        st_escs = {}
        t_escs = graph_time(torch, lambda: escs.escs_spmm(d["plan"], d["vals"], d["B"], d["C"], stream), stream,
                            reps=20, stats=st_escs)
        rp = torch.from_numpy(A.rowptr).to(dev["_device"])
        ci = torch.from_numpy(A.colidx).to(dev["_device"])
        Cs = torch.empty_like(d["C"])
        best, best_alg = None, None
        for alg in range(4):
            h = bl.bl_cusparse_create(A.m, A.k, A.nnz, n, rp.data_ptr(), ci.data_ptr(),
                                      d["vals"].data_ptr(), d["B"].data_ptr(), Cs.data_ptr(), alg, sp)
            if not h:
                continue
            try:
                t = graph_time(torch, lambda: bl.bl_cusparse_run(h, sp), stream)
            except Exception:
                t = None
            bl.bl_cusparse_destroy(h)
            if t and (best is None or t < best):
                best, best_alg = t, alg
        Ad = torch.from_numpy(A.dense()).to(dev["_device"])
        Cd = torch.empty_like(d["C"])
        t_cublas = graph_time(torch, lambda: bl.bl_cublas_sgemm(cub, A.m, n, A.k, Ad.data_ptr(), d["B"].data_ptr(), Cd.data_ptr(), 0, sp), stream)
        t_tf32 = graph_time(torch, lambda: bl.bl_cublas_sgemm(cub, A.m, n, A.k, Ad.data_ptr(), d["B"].data_ptr(), Cd.data_ptr(), 1, sp), stream)
        del Ad
        inf = d["plan"].info
        rows.append({"case": p.name, "escs_us": 1e3 * t_escs, "escs_us_min": 1e3 * st_escs["min"],
                     "escs_us_p90": 1e3 * st_escs["p90"],
                     "plan": {k: inf[k] for k in ("h", "T", "cta_warps", "ufk", "colf", "n_tiles", "n_heavy", "G")},
                     "cusparse_us": None if best is None else 1e3 * best, "cusparse_alg": best_alg,
                     "cublas_us": 1e3 * t_cublas, "cublas_tf32_us": 1e3 * t_tf32,
                     "gflops_escs": p.flops / (t_escs * 1e-3) / 1e9})
    bl.bl_cublas_destroy(cub)
    out = {
        "protocol": "hot L2, CUDA graph of R calls (R = clamp(2 ms / t, 10, 1000)) replayed 20x for escs, 11x for the baselines; median (paper P:675 warm cache); escs min and p90 per case",
        "geomean_speedup_vs_cusparse": geomean([r["cusparse_us"] / r["escs_us"] for r in rows if r["cusparse_us"]]),
        "geomean_speedup_vs_cublas": geomean([r["cublas_us"] / r["escs_us"] for r in rows]),
        "geomean_speedup_vs_cublas_tf32": geomean([r["cublas_tf32_us"] / r["escs_us"] for r in rows]),
        "pct_faster_than_cusparse": 100.0 * np.mean([r["cusparse_us"] is not None and r["escs_us"] < r["cusparse_us"] for r in rows]),
        "pct_faster_than_cublas": 100.0 * np.mean([r["escs_us"] < r["cublas_us"] for r in rows]),
        "cases": len(rows),
        "paper_context": "A100: 1.84x vs cuBLAS, 2.27x vs cuSPARSE (abstract P:31); Table 1 geomeans 1.47x / 1.74x",
    }
    return out, rows


def run_escs(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU (LOCAL_RANK); ESCS_BENCH_BACKEND=gloo lets a 1-GPU box
    # exercise the N > 1 control flow with several ranks sharing the device
    backend = os.environ.get("ESCS_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)

    from paper_2506_15174_b200 import escs, shard, synth

    problems, desc = workload(args.workload)
    # N > 1: a suite of independent problems is partitioned over ranks (LPT by
    # flops, no collective); a single large problem is row-block sharded with
    # B replicated.  N = 1: every problem whole.
    mode = args.shard
    if mode == "auto":
        mode = "problems" if len(problems) >= 2 * world else "rows"
    if world > 1 and mode == "problems":
        mine = shard.partition_problems([p.flops for p in problems], world)[rank]
        sharding = f"problems (LPT by flops) x{world}"
    else:
        mine = list(range(len(problems)))
        sharding = f"row-block x{world}"
    dev = {"_device": device}
    want_tp = bool(args.autotune and args.tp_plans and args.streams > 1 and len(mine) > 1)
    shard_problems = []
    plan_s = 0.0
    plan_info = []
    plan_info_tp = []
    for idx in mine:
        p = problems[idx]
        t0 = time.perf_counter()
        tune = {"autotune": 1} if args.autotune else {}
        if mode == "problems":
            A = p.A
            pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, p.bcols, **tune)
        else:
            A, pl = shard.plan_shard(p.A, p.bcols, world, rank, **tune)
        # throughput-objective plans (autotune = 2) for the multi-stream step:
        # the latency-tuned plan of a layer alone tends to fill every SM, which
        # starves the layers co-running on the other streams
        pl_tp = None
        if want_tp:
            if mode == "problems":
                pl_tp = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, p.bcols, autotune=2)
            else:
                pl_tp = shard.plan_shard(p.A, p.bcols, world, rank, autotune=2)[1]
        plan_s += time.perf_counter() - t0
        info = pl.info
        plan_info.append(info)
        plan_info_tp.append(pl_tp.info if pl_tp is not None else None)
        d = {"plan": pl, "plan_tp": pl_tp or pl, "A": A,
             "vals": torch.from_numpy(A.vals).to(device) if A.nnz else torch.zeros(1, device=device),
             "B": torch.from_numpy(p.B).to(device),
             "C": torch.empty((A.m, p.bcols), dtype=torch.float32, device=device),
             "flops": 2 * A.nnz * p.bcols,
             "bytes": 8 * A.nnz + 4 * (A.m + 1) + 4 * A.k * p.bcols + 4 * A.m * p.bcols,
             "gather_bytes": 4 * p.bcols * info["G"]}
        dev[p.name] = d
        shard_problems.append((p, d))
    flush = torch.empty(L2_FLUSH_BYTES // 4 if not args.hot_l2 else 4, dtype=torch.float32, device=device)
    # all work on one non-default stream (graph capture needs a non-default stream)
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)

    # --streams S > 1: the independent problems of a suite run on S streams
    # (LPT by flops), forked from and joined back into the timed stream, so
    # small latency-bound layers overlap on the SMs (the suite analogue of the
    # problem partition across ranks).  Each stream chains its launches with PDL.
    nstreams = max(1, min(args.streams, len(shard_problems)))
    lanes = [stream] + [torch.cuda.Stream(device) for _ in range(nstreams - 1)]
    groups = shard.partition_problems([d["flops"] for _, d in shard_problems], nstreams)
    owner = {i: g for g, idx in enumerate(groups) for i in idx}
    # multi-stream issue order: heaviest problems first (LPT list order), so
    # the long layers start at once and the short ones fill in behind them
    issue = (sorted(range(len(shard_problems)), key=lambda i: (-shard_problems[i][1]["flops"], i))
             if args.issue_order == "lpt" else list(range(len(shard_problems))))

    # --group: each stream's problems go through ONE escs_spmm_group call (one
    # launch per kernel instance, <= 32 problems each, instead of one per problem)
    grouped = None
    group_launches = len(shard_problems)
    if args.group:
        grouped = [escs.Group([shard_problems[i][1]["plan_tp"] for i in idx],
                              [shard_problems[i][1]["vals"] for i in idx],
                              [shard_problems[i][1]["B"] for i in idx],
                              [shard_problems[i][1]["C"] for i in idx]) for idx in groups]
        group_launches = 0
        for idx in groups:           # launches per call, as escs_spmm_group buckets them
            keys = {}
            for i in idx:
                inf = shard_problems[i][1]["plan_tp"].info
                if inf["h"] == 1 and inf["variant"] == 1:
                    key = (inf["bcols"], inf["colf"], inf["ufk"], inf["cta_warps"])
                    keys[key] = keys.get(key, 0) + 1
                else:
                    group_launches += 1
            group_launches += sum(-(-c // 32) for c in keys.values())

    def step(per_launch=None, serial=False):
        if serial:      # every launch on the timed stream (the 1-stream figure)
            for i, (p, d) in enumerate(shard_problems):
                if per_launch is not None:
                    per_launch[i][0].record(stream)
                escs.escs_spmm(d["plan"], d["vals"], d["B"], d["C"], stream)
                if per_launch is not None:
                    per_launch[i][1].record(stream)
            return
        if nstreams > 1:
            fork = torch.cuda.Event()
            fork.record(stream)
            for s_ in lanes[1:]:
                s_.wait_event(fork)
        if grouped:
            for g, st in zip(grouped, lanes):
                g(stream=st)
        else:
            for i in issue:
                p, d = shard_problems[i]
                st = lanes[owner[i]]
                if per_launch is not None:
                    per_launch[i][0].record(st)
                escs.escs_spmm(d["plan_tp"], d["vals"], d["B"], d["C"], st)
                if per_launch is not None:
                    per_launch[i][1].record(st)
        for s_ in lanes[1:]:
            j = torch.cuda.Event()
            j.record(s_)
            stream.wait_event(j)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up
    for _ in range(args.warmup):
        step()
    barrier()

    nprob = len(shard_problems)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    sleep_cycles = int(2e6 + 4e4 * nprob)

    # ---- timed: step events only (value)
    starts, ends = [ev() for _ in range(args.steps)], [ev() for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.nvtx.range_push("bench_timed")   # ncu --nvtx-include bench_timed/
        for s in range(args.steps):
            flush.zero_()
            torch.cuda._sleep(sleep_cycles)
            starts[s].record(stream)
            step()
            ends[s].record(stream)
        torch.cuda.nvtx.range_pop()
        barrier()
        # ---- the same steps with every launch on one stream (reported beside value)
        serial_ms = None
        if nstreams > 1:
            s0, s1 = [ev() for _ in range(args.steps)], [ev() for _ in range(args.steps)]
            for s in range(args.steps):
                flush.zero_()
                torch.cuda._sleep(sleep_cycles)
                s0[s].record(stream)
                step(serial=True)
                s1[s].record(stream)
            barrier()
            serial_ms = sum(a.elapsed_time(b) for a, b in zip(s0, s1))
        # ---- timed again with per-launch events (kernel durations for the roofline;
        # one stream, so each duration is the kernel alone)
        pl_ev = [[[ev(), ev()] for _ in range(nprob)] for _ in range(args.steps)]
        for s in range(args.steps):
            flush.zero_()
            torch.cuda._sleep(sleep_cycles)
            step(pl_ev[s], serial=True)   # kernels alone, like the probe below
        barrier()
    # ---- gather probe: same walk and B-row loads, no values/FMAs (t_probe)
    probe_ms = None
    if all(d["plan"].info["variant"] == 1 for _, d in shard_problems):
        sinks = [torch.empty(d["plan"].info["n_tiles"] * 32 * d["plan"].info["cta_warps"],
                             device=device) for _, d in shard_problems]
        pr_ev = [[[ev(), ev()] for _ in range(nprob)] for _ in range(args.steps)]
        for s_ in range(args.steps):
            flush.zero_()
            torch.cuda._sleep(sleep_cycles)
            for i, (p, d) in enumerate(shard_problems):
                pr_ev[s_][i][0].record(stream)
                escs.escs_gather_probe(d["plan"], d["B"], sinks[i], stream)
                pr_ev[s_][i][1].record(stream)
        barrier()
        probe_ms = float(sum(a.elapsed_time(b) for row in pr_ev for a, b in row))
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total_ms = sum(step_ms)
    kern_ms = np.array([[a.elapsed_time(b) for a, b in pl_ev[s]] for s in range(args.steps)])
    kern_ms_sum = float(kern_ms.sum())

    # ---- e2e: host buffers through the public API, copies inside the timed region.
    # The step's inputs (every layer's values and B) sit in one pinned host
    # buffer and its outputs land in one pinned host buffer; the step is cut
    # into --e2e-chunks chunks of layers pipelined over three streams (H2D of
    # chunk j+1 overlaps the SpMMs of chunk j; D2H of chunk j follows its
    # SpMMs on its own stream, overlapping later H2D and SpMMs).
    sizes_in = [(d["A"].nnz, p.B.size) for p, d in shard_problems]
    off_in, tot_in = [], 0
    for nv, nb in sizes_in:
        off_in.append(tot_in)
        tot_in += (max(nv, 1) + 3) // 4 * 4 + nb   # 16-byte aligned B views
    off_out, tot_out = [], 0
    for _, d in shard_problems:
        off_out.append(tot_out)
        tot_out += d["C"].numel()
    vpad = [(max(nv, 1) + 3) // 4 * 4 for nv, _ in sizes_in]
    h_in = torch.zeros(tot_in, dtype=torch.float32).pin_memory()
    h_out = torch.empty(tot_out, dtype=torch.float32).pin_memory()
    for i, (p, d) in enumerate(shard_problems):
        nv, nb = sizes_in[i]
        if nv:
            h_in[off_in[i]:off_in[i] + nv] = torch.from_numpy(d["A"].vals)
        h_in[off_in[i] + vpad[i]:off_in[i] + vpad[i] + nb] = torch.from_numpy(p.B.ravel())
    d_in = torch.empty(tot_in, dtype=torch.float32, device=device)
    d_out = torch.empty(tot_out, dtype=torch.float32, device=device)
    nchunk = min(args.e2e_chunks, nprob)
    # equal layer counts per chunk (measured: 880 GFLOP/s vs 785 with chunks
    # balanced by bytes -- a small first chunk starts the pipeline sooner)
    bounds = [(c * nprob) // nchunk for c in range(nchunk + 1)]
    copy_s = torch.cuda.Stream(device)
    out_s = torch.cuda.Stream(device)
    h2d = 4 * tot_in
    d2h = 4 * tot_out

    def e2e_step():
        evs = []
        for c in range(nchunk):            # H2D of every chunk on the copy stream
            a, b = bounds[c], bounds[c + 1]
            lo, hi = off_in[a], (off_in[b] if b < nprob else tot_in)
            copy_s.wait_stream(stream)
            with torch.cuda.stream(copy_s):
                d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
            e = torch.cuda.Event()
            e.record(copy_s)
            evs.append(e)
        for c in range(nchunk):            # SpMMs on the main stream, then D2H of the chunk
            stream.wait_event(evs[c])
            a, b = bounds[c], bounds[c + 1]
            for i in range(a, b):
                p, d = shard_problems[i]
                nv, nb = sizes_in[i]
                v = d_in[off_in[i]:off_in[i] + vpad[i]]
                Bv = d_in[off_in[i] + vpad[i]:off_in[i] + vpad[i] + nb]
                Cv = d_out[off_out[i]:off_out[i] + d["C"].numel()]
                escs.escs_spmm(d["plan"], v, Bv, Cv, stream)
            lo, hi = off_out[a], (off_out[b] if b < nprob else tot_out)
            out_s.wait_stream(stream)
            with torch.cuda.stream(out_s):         # D2H on its own engine/stream
                h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
        stream.wait_stream(out_s)

    if nprob == 1 and args.e2e_chunks > 1 and shard_problems[0][1]["A"].m >= 8 * args.e2e_chunks:
        # one large problem: pipeline by row blocks (one escs plan per block,
        # built once, outside the timed region).  H2D of B first, then each
        # block's values (contiguous in CSR order) while earlier blocks compute;
        # each block's C rows go back as soon as they are done.
        p0, d0 = shard_problems[0]
        A0, n0 = d0["A"], p0.bcols
        E = args.e2e_chunks
        blocks = []
        for r in range(E):
            r0, r1 = synth.shard_bounds(A0.m, E, r)
            S = synth.row_block(A0, r0, r1)
            tune = {"autotune": 1} if args.autotune and S.nnz <= 8_000_000 else {}
            pl = escs.escs_plan_ex(S.m, S.k, S.nnz, S.rowptr, S.colidx, n0, **tune)
            blocks.append((pl, int(A0.rowptr[r0]), S.nnz, r0, r1))
        bpad = (p0.B.size + 3) // 4 * 4
        h_in = torch.empty(bpad + max(A0.nnz, 1), dtype=torch.float32).pin_memory()
        h_in[:p0.B.size] = torch.from_numpy(p0.B.ravel())
        if A0.nnz:
            h_in[bpad:bpad + A0.nnz] = torch.from_numpy(A0.vals)
        h_out = torch.empty(A0.m * n0, dtype=torch.float32).pin_memory()
        d_in = torch.empty_like(h_in, device=device)
        d_out = torch.empty(A0.m * n0, dtype=torch.float32, device=device)
        h2d, d2h = 4 * (p0.B.size + A0.nnz), 4 * A0.m * n0
        Bv = d_in[:p0.B.size]

        def e2e_step():
            evs = []
            copy_s.wait_stream(stream)
            with torch.cuda.stream(copy_s):
                d_in[:p0.B.size].copy_(h_in[:p0.B.size], non_blocking=True)
                for pl, v0, nv, r0, r1 in blocks:
                    d_in[bpad + v0:bpad + v0 + nv].copy_(h_in[bpad + v0:bpad + v0 + nv], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(copy_s)
                    evs.append(e)
            for (pl, v0, nv, r0, r1), e in zip(blocks, evs):
                stream.wait_event(e)
                vv = d_in[bpad + v0:bpad + v0 + max(nv, 1)]
                escs.escs_spmm(pl, vv, Bv, d_out[r0 * n0:r1 * n0], stream)
                out_s.wait_stream(stream)
                with torch.cuda.stream(out_s):
                    h_out[r0 * n0:r1 * n0].copy_(d_out[r0 * n0:r1 * n0], non_blocking=True)
            stream.wait_stream(out_s)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier()
    es, ee = [ev() for _ in range(args.steps)], [ev() for _ in range(args.steps)]
    for s in range(args.steps):
        flush.zero_()
        torch.cuda._sleep(sleep_cycles)
        es[s].record(stream)
        e2e_step()
        ee[s].record(stream)
    barrier()
    e2e_ms = sum(a.elapsed_time(b) for a, b in zip(es, ee))
    # the copies alone (same buffers, same chunking): the PCIe floor of e2e
    ca, cb = ev(), ev()
    ca.record(stream)
    for _ in range(args.steps):
        with torch.cuda.stream(copy_s):
            copy_s.wait_stream(stream)
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(out_s):
            out_s.wait_stream(stream)
            h_out.copy_(d_out, non_blocking=True)
        stream.wait_stream(copy_s)
        stream.wait_stream(out_s)
    cb.record(stream)
    torch.cuda.synchronize(device)
    copy_ms = ca.elapsed_time(cb) / args.steps

    # ---- optional all-gather of C (NCCL), timed separately (not on the hot path)
    allgather_ms = None
    if world > 1 and args.allgather and mode == "rows":
        ga, gb = ev(), ev()
        barrier()
        ga.record(stream)
        for p, d in shard_problems:
            shard.all_gather_rows(d["C"], p.A.m, world)
        gb.record(stream)
        barrier()
        allgather_ms = shard.max_over_ranks([ga.elapsed_time(gb)], device)[0]
    # ---- SpMM fused with the all-gather (NEXT f1): escs_spmm_scatter stores
    # each C row into every rank's symmetric-memory C (NVLink P2P / NVLS
    # multicast); timed per step against SpMM + NCCL all-gather
    fused = None
    if world > 1 and args.allgather and mode == "rows" and backend == "nccl":
        try:
            fgs = [shard.FusedGather(p.A.m, p.bcols) for p, _ in shard_problems]
            def fused_step():
                for fg, (p, d) in zip(fgs, shard_problems):
                    fg.run(d["plan"], d["vals"], d["B"], stream)
            def split_step():
                for p, d in shard_problems:
                    escs.escs_spmm(d["plan"], d["vals"], d["B"], d["C"], stream)
                    shard.all_gather_rows(d["C"], p.A.m, world)
            fused = {"mode": fgs[0].mode}
            for name, fn in (("fused_ms_per_step", fused_step), ("spmm_then_nccl_ms_per_step", split_step)):
                for _ in range(args.warmup):
                    fn()
                fa, fb = ev(), ev()
                barrier()
                fa.record(stream)
                for _ in range(args.steps):
                    fn()
                fb.record(stream)
                barrier()
                fused[name] = shard.max_over_ranks([fa.elapsed_time(fb) / args.steps], device)[0]
        except Exception as e:            # symmetric memory unavailable on this box
            fused = {"unavailable": str(e)[:200]}

    # ---- reduce over ranks: flops SUM, times MAX
    my_flops = sum(d["flops"] for _, d in shard_problems)
    my_bytes = sum(d["bytes"] for _, d in shard_problems)
    total_ms, e2e_ms, kern_ms_sum, serial_ms = shard.max_over_ranks(
        [total_ms, e2e_ms, kern_ms_sum, serial_ms or 0.0], device)
    flops_all, bytes_all = shard.sum_over_ranks([my_flops, my_bytes], device)

    result = None
    if rank == 0:
        hbm, peak_src, mp = peaks()
        K = args.steps
        value = flops_all * K / (total_ms * 1e-3) / 1e9
        # roofline of the (only) kernel: compulsory bytes per launch / launch duration
        achieved = my_bytes * K / (kern_ms.sum() * 1e-3) / 1e9
        gather = sum(d["gather_bytes"] for _, d in shard_problems) * K / (total_ms * 1e-3) / 1e9
        per_prob = kern_ms.mean(axis=0)
        dom = int(np.argmax(per_prob))
        clocks = clk.summary()
        traffic, traffic_src = committed_traffic(args.workload) if world == 1 else (None, None)
        n_sm = torch.cuda.get_device_properties(device).multi_processor_count
        gather_derived = n_sm * 64.0 * float(mp.get("sm_max_mhz", 1965.0)) * 1e6 / 1e9
        try:
            gather_peak, gather_src = gather_ceiling(torch, device, stream, n_sm), (
                "measured in this run: bl_gather_peak (libescs_bench.so) gathers pseudo-random 512-byte "
                "rows of a 64 MiB L2-resident B, no index loads / values / FMAs, best of 6 lane maps")
        except (OSError, AssertionError):
            gather_peak, gather_src = gather_derived, "derived: SMs x 64 B/clk x max SM clock"
        step_bytes_per_s = my_bytes * K / (total_ms * 1e-3) / 1e9
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "problems": len(problems), "sharding": sharding,
                       "streams": nstreams,
                       "grouped": bool(args.group),
                       "l2": ("flushed before every step (256 MiB write); each problem touched once per step"
                              if not args.hot_l2 else "NOT flushed (--hot-l2 diagnostic, not a bench value)"),
                       "plans": (("autotuned at plan time (escs_params.autotune: timed T / tile width / UFk candidates); "
                                  + ("the multi-stream step (value) runs throughput-objective plans (autotune=2: candidates "
                                     "timed as 8 concurrent launch chains on 8 streams), serial / per-launch / per-case figures "
                                     "the latency-objective plans (autotune=1)" if want_tp else "latency objective (autotune=1)"))
                                 if args.autotune else "parameter table (escs_plan defaults)"),
                       "plan": {k: plan_info[dom][k] for k in ("h", "T", "cta_warps", "ufk", "colf", "variant")},
                       "plan_throughput": ({k: plan_info_tp[dom][k] for k in ("h", "T", "cta_warps", "ufk", "colf", "variant")}
                                           if plan_info_tp[dom] is not None else None)},
            "roofline": {"bound": "hbm", "achieved": step_bytes_per_s, "peak": hbm, "unit": "GB/s",
                         "frac": step_bytes_per_s / hbm, "traffic": traffic,
                         "achieved_how": ("algorithmic bytes of the step / timed step (CUDA events on the "
                                          "launching streams; the timed region holds only escs_spmm launches, "
                                          "back to back with PDL on each of config.streams streams)"),
                         "achieved_per_launch_bracketed": achieved,
                         "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": my_bytes / nprob,
                         "peak_source": peak_src,
                         "algorithmic_bytes": "8*nnz + 4*(m+1) + 4*k*bCols + 4*m*bCols per launch (CSR A, B, C once; SURVEY 8(d))",
                         "kernel": "escs_spmm (esc_spmm_kernel), all launches of the step",
                         "kernel_ms_per_step": float(kern_ms.sum() / K),
                         "kernel_ms_how": "sum of per-launch CUDA-event durations, launches on one stream (each kernel alone)",
                         "gather_GBps": gather,
                         "gather_bytes": "4*bCols per gcol (one B row per (panel,column) pair)",
                         "gather_roofline": {
                             "achieved": gather, "unit": "GB/s",
                             "peak": gather_peak, "frac": gather / gather_peak,
                             "peak_source": gather_src,
                             "derived_64B_per_clk": gather_derived},
                         "attainable": None if probe_ms is None else {
                             "probe_ms_per_step": probe_ms / K,
                             "frac": probe_ms / float(kern_ms.sum()),
                             "what": "t_probe / t_kernel: escs_gather_probe runs the same item walk and B-row gathers without values or FMAs (measured gather ceiling of this plan)"}},
            "gpu_launches": group_launches * K,   # this rank's kernel launches in the timed region
            "clocks": clocks,
            "e2e": {"value": flops_all * K / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "copies_only_ms_per_step": copy_ms,
                    "copy_floor": (f"{(h2d + d2h) / (copy_ms * 1e-3) / 1e9:.1f} GB/s host<->device "
                                   f"(H2D and D2H concurrent); e2e is {e2e_ms / K / copy_ms:.2f}x "
                                   "the copies alone")},
            "plan_seconds": plan_s,
        }
        if nstreams > 1:
            result["serial"] = {"value": flops_all * K / (serial_ms * 1e-3) / 1e9, "unit": UNIT,
                                "ms_per_step": serial_ms / K,
                                "what": "same steps, every escs_spmm on one stream (PDL chain)"}
        if allgather_ms is not None:
            result["allgather_ms_per_step"] = allgather_ms
        if fused is not None:
            result["fused_allgather"] = fused
        if world == 1 and not args.no_cpu:
            v, reps, secs, thr = oracle_time(problems, budget_s=args.cpu_budget)
            result["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle",
                                      "sample": f"whole workload x{reps} ({secs:.1f} s), fp64 C oracle"}
            # one-time planning costs (the paper excludes its dataTransformer from
            # SpMM time): escs_plan (h-way merge, threaded, incl. autotuning)
            # vs the oracle's dense-scan partitioner (O(m*k) per problem)
            if sum(p.A.m * p.A.k for p in problems) <= 2e9:
                import oracle
                t0 = time.perf_counter()
                for p, d in shard_problems:
                    inf = d["plan"].info
                    oracle.partition(p.A.m, p.A.k, p.A.rowptr, p.A.colidx, inf["h"], inf["T"], p.bcols)
                result["planning"] = {"escs_plan_s": plan_s,
                                      "oracle_partition_s": time.perf_counter() - t0,
                                      "what": "one-time host planning for the whole workload (not in value)"}
        if world == 1 and not args.no_compare:
            summ, rows = compare_baselines(torch, problems, dev, stream)
            result["baselines"] = summ
            if args.cases_out:
                with open(args.cases_out, "w") as f:
                    json.dump(rows, f, indent=1)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if result is not None:
        print(json.dumps(result), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="escs", choices=["escs", "reference"])
    ap.add_argument("--workload", default="suite")
    ap.add_argument("--no-compare", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--hot-l2", action="store_true",
                    help="diagnostic only: skip the L2 flush between steps (not a bench value)")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--group", type=int, default=0,
                    help="1: each stream's problems in one escs_spmm_group call (grouped launches)")
    ap.add_argument("--issue-order", default="lpt", choices=("lpt", "index"),
                    help="multi-stream step: launch problems heaviest-first (lpt) or in suite order")
    ap.add_argument("--streams", type=int, default=16,
                    help="suite: run the independent problems on this many streams (LPT by flops)")
    ap.add_argument("--cases-out", default=None)
    ap.add_argument("--no-tp-plans", dest="tp_plans", action="store_false",
                    help="run the multi-stream step on the latency-tuned plans too (no autotune=2 plans)")
    ap.add_argument("--no-autotune", dest="autotune", action="store_false",
                    help="plan with the parameter table only (default: plan-time autotuning)")
    ap.add_argument("--shard", default="auto", choices=["auto", "rows", "problems"],
                    help="N>1: partition a suite by problems or row-block shard every problem")
    ap.add_argument("--e2e-chunks", type=int, default=8,
                    help="e2e: copy/compute pipeline depth (chunks of layers per step)")
    ap.add_argument("--allgather", action="store_true",
                    help="N>1: also time the optional NCCL all-gather of C (not on the hot path)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_escs(args)


if __name__ == "__main__":
    sys.exit(main())
