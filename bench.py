#!/usr/bin/env python3
"""Benchmark: batched FP64 GEMM (BASELINE.json metric) on 1..N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl lrb|reference]

A step is one pass of the hot path over the rank's batch, inputs resident in
HBM (generated on device, untimed). Default workload: BASELINE configs[1]
(cfg2, low-rank expansion U V^T, 4096 items of 512x32 * (512x32)^T), the
config the metric is quoted on. Under torchrun each rank owns one GPU and a
contiguous item range; there is no data-path collective (items are
independent): only a barrier and a max-over-ranks of the device time.

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_PEAK_FALLBACK = 6553.6  # GB/s
FP64_PEAK_MEASURED = 36.9   # TFLOP/s, tools/microbench/fp64_peaks.cu on this pool (DMMA == DFMA)


# ------------------------------------------------------------------ helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm, src = HBM_PEAK_FALLBACK, "fallback (B200_PROFILING.md)"
    try:
        with open(p) as f:
            d = json.load(f)
        hbm = float(d.get("hbm_gbs", hbm))
        src = "MEASURED_PEAKS.json"
    except Exception:
        pass
    fp64, fsrc = FP64_PEAK_MEASURED, "measured: tools/microbench/fp64_peaks.cu (profiles/fp64_peaks_r01.jsonl)"
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peaks_r01.jsonl")) as f:
            vals = [json.loads(l) for l in f if l.strip().startswith("{")]
        best = max(v["tflops"] for v in vals if v.get("probe", "").startswith(("dmma", "dfma")))
        fp64 = float(best)
    except Exception:
        pass
    return hbm, src, fp64, fsrc


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region"""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # the only collectives are a barrier and a max of per-rank device time:
        # gloo on host scalars keeps torch off the GPU entirely
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pg = dist
    return world, rank, local, pg


def barrier(pg):
    if pg is not None:
        pg.barrier()


def all_max(pg, x: float) -> float:
    if pg is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def all_sum(pg, x: float) -> float:
    if pg is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


# ----------------------------------------------------------- workload slice
def rank_items(w, world, rank):
    """(first global item, count) of this rank. cfg5 is the whole-box batch
    split across ranks (strong scaling); the others keep the BASELINE batch per
    GPU and index items globally (weak scaling)."""
    from paper_2311_07602_b200 import shard_plan

    if w.name == "cfg5":
        b = shard_plan(w.batch, world)
        return b[rank], b[rank + 1] - b[rank], "strong"
    return rank * w.batch, w.batch, "weak"


def traffic_from_profiles(config_name: str):
    """dram bytes per launch of the top kernel from the committed ncu summary"""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(config_name)
    except Exception:
        return None


# ------------------------------------------------------------- CPU baseline
def cpu_sample_run(w, items, threads):
    """time the reference binary (oracle/_ref, else the C restatement) on a
    bounded sample of the workload's items; returns (seconds, flops, kind)"""
    import numpy as np

    import oracle as O
    from paper_2311_07602_b200 import workloads as W

    n = len(items)
    first = items[0]
    if isinstance(w, W.Strided):
        A = O.fill_uniform(w.a_rows, w.a_cols, w.lda, w.sA, n, w.seed, W.ROLE_A, first)
        B = O.fill_uniform(w.b_rows, w.b_cols, w.ldb, w.sB, n, w.seed, W.ROLE_B, first)
        Cm = np.zeros(w.sC * n)
        t0 = time.perf_counter()
        if O.ref_available() and w.order == "R" and w.opA == "N" and w.opB == "N":
            # the reference's own row-major call, item by item
            O.ref_rowmajor_batched(A, B, Cm, w.m, w.k, w.n, 0, n, threads=threads)
            kind = "reference"
        elif O.ref_available() and w.order == "C":
            O.ref_dgemm_colmajor(w.opA, w.opB, w.m, w.n, w.k, 0, A, w.lda, w.sA, B, w.ldb, w.sB,
                                 Cm, w.ldc, w.sC, n, threads=threads)
            kind = "reference"
        else:
            O.dgemm_strided(w.order, w.opA, w.opB, w.m, w.n, w.k, 0.0, A, w.lda, w.sA, B, w.ldb,
                            w.sB, Cm, w.ldc, w.sC, n, threads=threads, mode=O.REF_COMPILED)
            kind = "port"
        dt = time.perf_counter() - t0
        return dt, w.item_flops() * n, w.item_bytes() * n, kind
    # variable-size
    ids = items
    As = [O.fill_uniform(w.bs[i], w.bs[i], w.bs[i], 0, 1, w.seed, W.ROLE_A, i) for i in ids]
    Bs = [O.fill_uniform(w.bs[i], w.rs[i], w.bs[i], 0, 1, w.seed, W.ROLE_B, i) for i in ids]
    Cs = [np.zeros(w.bs[i] * w.rs[i]) for i in ids]
    ms = [w.bs[i] for i in ids]
    ns = [w.rs[i] for i in ids]
    t0 = time.perf_counter()
    if O.ref_available():
        O.ref_dgemm_colmajor_ptr("N", "N", ms, ns, ms, As, ms, Bs, ms, Cs, ms, 0, threads=threads)
        kind = "reference"
    else:
        O.dgemm_ptr("C", "N", "N", ms, ns, ms, As, ms, Bs, ms, Cs, ms, 0.0, threads=threads,
                    mode=O.REF_COMPILED)
        kind = "port"
    dt = time.perf_counter() - t0
    return dt, w.flops(ids), w.bytes(ids), kind


def pick_sample(w, threads, target_s):
    """deterministic bounded sample: calibrate one item, then ~target_s of CPU work"""
    from paper_2311_07602_b200 import workloads as W

    dt1, fl1, _, _ = cpu_sample_run(w, [0], 1)
    per_item = max(dt1, 1e-6)
    total_batch = w.batch
    n = int(max(threads, min(total_batch, threads * max(1, int(target_s / per_item)))))
    n = min(n, total_batch)
    step = max(1, total_batch // n)
    items = list(range(0, step * n, step))[:n]
    if isinstance(w, W.Strided):
        items = list(range(items[0], items[0] + n))  # contiguous for the strided API
    return items


def run_reference_arm(args, w, world, rank):
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    threads = os.cpu_count() or 1
    items = pick_sample(w, threads, args.ref_seconds)
    for _ in range(max(0, args.warmup_ref)):
        cpu_sample_run(w, items, threads)
    times, fl, by, kind = [], 0.0, 0.0, "reference"
    for _ in range(args.steps):
        dt, fl, by, kind = cpu_sample_run(w, items, threads)
        times.append(dt)
    t = statistics.median(times)
    gflops = fl / t / 1e9
    sample = (f"{len(items)} of {w.batch} items of {w.name} per step "
              f"(items {items[0]}..{items[-1]}), std::thread contiguous split like "
              f"naive_multiply_batch; value extrapolates per-item rate to the workload")
    line = {
        "metric": "batched FP64 GFLOP/s", "value": round(gflops, 3), "unit": "GFLOP/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (counter RNG, uniform[-1,1))",
        "config": dict(w.describe(), sample_items=len(items)),
        "hbm_gbs": None,
        "cpu_baseline": {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": threads,
                         "kind": kind, "sample": sample},
        "e2e": {"value": round(gflops, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def alloc_inputs(ctx, w, first, count, shard=None):
    from paper_2311_07602_b200 import workloads as W

    A = ctx.empty(w.sA * count)
    B = ctx.empty(w.sB * count)
    Cd = ctx.empty(w.sC * count)
    ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, count, w.seed, W.ROLE_A, first)
    ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, count, w.seed, W.ROLE_B, first)
    ctx.synchronize()
    return A, B, Cd


def gemm(ctx, w, A, B, Cd, count, stream=None):
    ctx.dgemm_strided_batched(w.order, w.opA, w.opB, w.m, w.n, w.k, 0.0, A, w.lda, w.sA, B,
                              w.ldb, w.sB, Cd, w.ldc, w.sC, count, stream)


class VariableSlice:
    """cfg4 on one rank: arenas with 256-B aligned bases, a pointer-array plan"""

    def __init__(self, ctx, w, items):
        from paper_2311_07602_b200 import workloads as W

        self.items = items
        offs, (na, nb, nc) = W.variable_layout(w, items)
        self.arena = [ctx.malloc(na), ctx.malloc(nb), ctx.malloc(nc)]
        pa = [self.arena[0].ptr + o[0] for o in offs]
        pb = [self.arena[1].ptr + o[1] for o in offs]
        pc = [self.arena[2].ptr + o[2] for o in offs]
        bs = [w.bs[i] for i in items]
        rs = [w.rs[i] for i in items]
        # fill item by item with GLOBAL indices: contiguous runs keep it one call
        ctx.fill_uniform_ptr(pa, bs, bs, bs, w.seed, W.ROLE_A, items[0])
        ctx.fill_uniform_ptr(pb, bs, rs, bs, w.seed, W.ROLE_B, items[0])
        self.plan = ctx.ptr_plan("C", "N", "N", bs, rs, bs, pa, bs, pb, bs, pc, bs, 0.0)
        ctx.synchronize()


def run_gpu_arm_variable(args, w, world, rank, local, pg):
    from paper_2311_07602_b200 import Context, shard_plan

    hbm_peak, hbm_src, fp64_peak, fp64_src = load_peaks()
    ctx = Context(local)
    stream = ctx.stream()
    # weak scaling: every rank runs the full 8192-item cfg4 batch with its own
    # global item range (items rank*batch ..), drawn from the same seed stream
    base = rank * w.batch
    import copy

    wr = copy.copy(w)
    if base:
        wr = type(w)(w.name, w.batch * (rank + 1), w.seed)
    items = list(range(base, base + w.batch))
    vs = VariableSlice(ctx, wr, items)
    for _ in range(args.warmup):
        vs.plan.execute(stream)
    stream.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    barrier(pg)
    launches0 = ctx.launch_count
    t0, t1 = ctx.event(), ctx.event()
    t0.record(stream)
    for _ in range(args.steps):
        vs.plan.execute(stream)
    t1.record(stream)
    stream.synchronize()
    barrier(pg)
    clocks = sampler.stop()
    launches = ctx.launch_count - launches0
    ms_rank = t0.elapsed_ms(t1)
    ms_step = all_max(pg, ms_rank) / args.steps
    fl = wr.flops(items)
    by = wr.bytes(items)
    fl_all = all_sum(pg, fl)
    by_all = all_sum(pg, by)
    gflops = fl_all / (ms_step * 1e-3) / 1e9
    intensity = fl / by
    roof_t = min(fp64_peak * 1e12, intensity * hbm_peak * 1e9)
    achieved = fl / (ms_rank / args.steps * 1e-3)
    roof = {"bound": "tensor" if intensity * hbm_peak * 1e9 >= fp64_peak * 1e12 else "hbm",
            "achieved": round(achieved / 1e12, 3), "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": round(achieved / (fp64_peak * 1e12), 4),
            "roofline_frac": round(achieved / roof_t, 4), "traffic": None,
            "algorithmic": by, "kernel": "lrb_gemm_kernel<n8|n16|n32|n64> (ptr)",
            "kernel_ms": round(ms_rank / max(1, launches), 4),
            "peak_source": fp64_src}
    tr = traffic_from_profiles(w.name)
    if isinstance(tr, dict):
        roof["traffic"] = tr.get("dram_bytes_per_launch")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        sample = pick_sample(w, threads, args.ref_seconds)
        dt, sfl, _, kind = cpu_sample_run(w, sample, threads)
        cpu = {"value": round(sfl / dt / 1e9, 3), "unit": "GFLOP/s", "cores": threads,
               "kind": kind, "sample": f"{len(sample)} of {w.batch} cfg4 items ({dt:.1f} s)"}
    if rank == 0:
        cfg = dict(w.describe())
        cfg.update({"parallelism": f"shard{world} (independent items, no collective)",
                    "launches_per_step": vs.plan.launches,
                    "l2": "inputs larger than L2 (no flush)"})
        line = {
            "metric": "batched FP64 GFLOP/s", "value": round(gflops, 2), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device counter RNG, uniform[-1,1), BASELINE seeds)",
            "config": cfg, "hbm_gbs": round(by_all / (ms_step * 1e-3) / 1e9, 1),
            "roofline": roof, "cpu_baseline": cpu, "e2e": None, "clocks": clocks,
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def run_gpu_arm(args, w, world, rank, local, pg):
    from paper_2311_07602_b200 import Context, select, workloads as W

    if isinstance(w, W.Variable):
        return run_gpu_arm_variable(args, w, world, rank, local, pg)

    hbm_peak, hbm_src, fp64_peak, fp64_src = load_peaks()
    ctx = Context(local)
    stream = ctx.stream()
    first, count, scaling = rank_items(w, world, rank)

    # ---- device-resident inputs (chunked if the slice exceeds HBM)
    free, _ = ctx.mem_info()
    per_item = 8 * (w.sA + w.sB + w.sC)
    cap_items = max(1, int((free - (2 << 30)) // per_item))
    chunk = min(count, cap_items)
    nchunks = (count + chunk - 1) // chunk
    resident = nchunks == 1
    # a working set within 3x L2 (cfg1: 151 MB) rotates over identical copies
    # of its inputs and outputs, so no step finds the previous step's data in L2
    L2_BYTES = 132644864
    copies = 1
    if resident and per_item * count < 3 * L2_BYTES:
        copies = min(int(-(-3 * L2_BYTES // (per_item * count))),
                     max(1, int((free - (2 << 30)) // (per_item * count))))
    bufs = [alloc_inputs(ctx, w, first, chunk) for _ in range(copies)]
    A, B, Cd = bufs[0]
    rot = [0]

    def step():
        """one pass over this rank's items; returns device ms of the GEMM launches"""
        if resident:
            a, b, c = bufs[rot[0] % copies]
            rot[0] += 1
            gemm(ctx, w, a, b, c, count, stream)
            return None
        # chunked (cfg5 below 4 GPUs): regenerate each chunk (untimed), time GEMMs
        total = 0.0
        for c in range(nchunks):
            c0 = c * chunk
            cn = min(chunk, count - c0)
            ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, cn, w.seed, W.ROLE_A, first + c0,
                             stream)
            ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, cn, w.seed, W.ROLE_B, first + c0,
                             stream)
            e0.record(stream)
            gemm(ctx, w, A, B, Cd, cn, stream)
            e1.record(stream)
            stream.synchronize()
            total += e0.elapsed_ms(e1)
        return total

    e0, e1 = ctx.event(), ctx.event()
    for _ in range(args.warmup):
        step()
    stream.synchronize()

    # resident batches: the K timed steps are captured once as a CUDA graph
    # (lrb_graph_*) and replayed with one host call, so short steps (cfg1,
    # ~35 us) are not separated by host enqueue gaps
    graph = None
    if resident and not args.no_graph:
        with ctx.capture(stream) as cap:
            for _ in range(args.steps):
                step()
        graph = cap.graph

    # ---- timed region
    sampler = ClockSampler(local)
    sampler.start()
    barrier(pg)
    stream.synchronize()
    launches0 = ctx.launch_count
    t_start, t_end = ctx.event(), ctx.event()
    chunk_ms = 0.0
    t_start.record(stream)
    if graph is not None:
        graph.launch(stream)
    else:
        for _ in range(args.steps):
            r = step()
            if r is not None:
                chunk_ms += r
    t_end.record(stream)
    stream.synchronize()
    barrier(pg)
    clocks = sampler.stop()
    launches = ctx.launch_count - launches0
    ms_rank = t_start.elapsed_ms(t_end) if resident else chunk_ms
    if not resident:  # only GEMM launches count (fills between chunks are setup)
        launches = args.steps * nchunks
    ms_total = all_max(pg, ms_rank)
    ms_step = ms_total / args.steps
    items_all = all_sum(pg, float(count))
    flops_all = w.item_flops() * items_all
    bytes_all = w.item_bytes() * items_all
    gflops = flops_all / (ms_step * 1e-3) / 1e9
    gbs = bytes_all / (ms_step * 1e-3) / 1e9

    # ---- dominant kernel roofline (this rank, per launch)
    per_launch_ms = ms_rank / max(1, launches)
    # average items per launch (chunks may be unequal; algorithmic units per launch)
    launch_items = count / nchunks
    sel = select(w.order, w.opA, w.opB, w.m, w.n, w.k, chunk, ctx)
    intensity = w.item_flops() / w.item_bytes()
    fp64_bound = intensity >= (fp64_peak * 1e12) / (hbm_peak * 1e9)
    if fp64_bound:
        achieved = w.item_flops() * launch_items / (per_launch_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": round(achieved / fp64_peak, 4),
                "peak_source": fp64_src + " (FP64 DMMA; MEASURED_PEAKS.json has no FP64 figure)"}
    else:
        achieved = w.item_bytes() * launch_items / (per_launch_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "peak_source": hbm_src}
    tr = traffic_from_profiles(w.name)
    roof["traffic"] = tr.get("dram_bytes_per_launch") if isinstance(tr, dict) else None
    roof["algorithmic"] = w.item_bytes() * launch_items
    roof["kernel"] = ("lrb_panel_kernel<p256>" if sel["name"] == "p256" else
                      f"lrb_gemm_kernel<{sel['name']}>")
    roof["kernel_ms"] = round(per_launch_ms, 4)
    roof["roofline_frac"] = round(
        (w.item_flops() * launch_items / (per_launch_ms * 1e-3)) /
        min(fp64_peak * 1e12, intensity * hbm_peak * 1e9), 4)

    # ---- e2e through the host-buffer C-ABI (pinned host memory, copies timed)
    del A, B, Cd, bufs
    e2e = run_e2e(args, ctx, w, first, count, pg) if args.e2e_steps > 0 else None

    # ---- CPU baseline on rank 0 at N = 1
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        items = pick_sample(w, threads, args.ref_seconds)
        dt, fl, _, kind = cpu_sample_run(w, items, threads)
        cpu = {"value": round(fl / dt / 1e9, 3), "unit": "GFLOP/s", "cores": threads,
               "kind": kind,
               "sample": f"{len(items)} of {w.batch} items of {w.name} ({dt:.1f} s), per-item "
                         f"rate; std::thread contiguous split like naive_multiply_batch"}

    if rank == 0:
        cfg = dict(w.describe())
        cfg.update({"items_per_rank": count, "global_items": int(items_all),
                    "timed_launch": "CUDA graph of the K steps" if graph is not None
                    else "eager launches",
                    "parallelism": f"shard{world} (independent items, no collective)",
                    "kernel_variant": sel["name"],
                    "l2": (f"{copies} rotating copies of inputs+outputs "
                           f"({per_item * count * copies / 2**20:.0f} MiB) > 3x L2"
                           if copies > 1 else "inputs larger than L2 (no flush)"),
                    "chunks_per_step": nchunks})
        line = {
            "metric": "batched FP64 GFLOP/s", "value": round(gflops, 2), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device counter RNG, uniform[-1,1), BASELINE seeds)",
            "config": cfg, "hbm_gbs": round(gbs, 1), "roofline": roof, "cpu_baseline": cpu,
            "e2e": e2e, "clocks": clocks, "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def run_e2e(args, ctx, w, first, count, pg):
    """same metric through lrb_dgemm_strided_batched_host: pinned host inputs,
    H2D + kernels + D2H of the result inside the timed region"""
    # whole batch when it fits in 16 GiB of pinned host memory (cfg5's 288 GiB
    # does not: its e2e runs on the largest prefix that does)
    per_item = 8 * (w.sA + w.sB + w.sC)
    n = min(count, args.e2e_items) if args.e2e_items else min(count, (16 << 30) // per_item)
    A, B, _ = alloc_inputs(ctx, w, first, n)
    hA, hB, hC = ctx.pinned(w.sA * n), ctx.pinned(w.sB * n), ctx.pinned(w.sC * n)
    from paper_2311_07602_b200.lrbatch import _check, lib  # noqa

    _check(lib.lrb_memcpy_d2h(ctx._h, hA.ptr, A.ptr, hA.nbytes), ctx._h)
    _check(lib.lrb_memcpy_d2h(ctx._h, hB.ptr, B.ptr, hB.nbytes), ctx._h)
    del A, B

    def once():
        ctx.dgemm_strided_batched_host(w.order, w.opA, w.opB, w.m, w.n, w.k, 0.0, hA.array,
                                       w.lda, w.sA, hB.array, w.ldb, w.sB, hC.array, w.ldc, w.sC,
                                       n)

    once()
    barrier(pg)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        once()
    dt = (time.perf_counter() - t0) / args.e2e_steps
    dt = all_max(pg, dt)
    items_all = all_sum(pg, float(n))
    return {"value": round(w.item_flops() * items_all / dt / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(8 * (w.sA + w.sB) * n),
            "d2h_bytes_per_step": int(8 * w.sC * n), "items_per_rank": n,
            "ms_per_step": round(dt * 1e3, 2),
            "path": "lrb_dgemm_strided_batched_host (3-stream chunked H2D/kernel/D2H)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="lrb", choices=["lrb", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-items", type=int, default=0, help="0 = the rank's whole batch")
    ap.add_argument("--ref-seconds", type=float, default=4.0,
                    help="CPU work per reference-arm step / cpu_baseline sample")
    ap.add_argument("--warmup-ref", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the timed steps one by one instead of as a CUDA graph")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "lrb":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    from paper_2311_07602_b200 import workloads as W

    w = W.get(args.config)
    world, rank, local, pg = dist_setup()
    import bench_rows as R

    bench_mod = sys.modules[__name__]
    if isinstance(w, W.LowRank):
        if args.impl == "reference":
            R.run_lowrank_reference(args, w, world, rank, bench_mod)
        else:
            R.run_lowrank_gpu(args, w, world, rank, local, pg, bench_mod)
    elif isinstance(w, W.Blr):
        if args.impl == "reference":
            R.run_blr_reference(args, w, world, rank, bench_mod)
        else:
            R.run_blr_gpu(args, w, world, rank, local, pg, bench_mod)
    elif isinstance(w, (W.LrExpand, W.BlrDense)):
        if args.impl == "reference":
            R.run_expand_reference(args, w, world, rank, bench_mod)
        else:
            R.run_expand_gpu(args, w, world, rank, local, pg, bench_mod)
    elif args.impl == "reference":
        run_reference_arm(args, w, world, rank)
    else:
        run_gpu_arm(args, w, world, rank, local, pg)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
