#!/usr/bin/env python3
"""Benchmark: batched FP64 GEMM (BASELINE.json metric) on 1..N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl lrb|reference]
    python bench.py --gpus N --plan-only      # the shard plan only (no GPU)

A step is one pass of the hot path over the rank's items, inputs resident in
HBM (generated on device, untimed). Default workload: BASELINE configs[3]
(cfg4, 8192 variable-size pointer-array products A_i(b_i x b_i) B_i(b_i x r_i)),
the largest BASELINE config that fits one GPU (cfg5, the metric's 1/2/4/8-GPU
batch, is 288 GiB).

One process per GPU. Under torchrun the ranks come from RANK / LOCAL_RANK /
WORLD_SIZE; without torchrun, ``--gpus N`` (N > 1) launches the N ranks itself
(and fails when fewer than N GPUs are visible). Items are independent, so the
ranks exchange nothing on the data path: each takes its range from the shard
planner (lrb_shard_plan; cfg4 cut at equal cumulative per-item roofline time,
cfg5 split evenly, the others one BASELINE batch per GPU) and generates its
own items on device from global item indices. The only collectives are a
barrier and gathers of host scalars over gloo.

Timing: W untimed warm-up steps, then K steps, each one CUDA-graph replay
bracketed by CUDA events on the launching stream; a barrier and a device
synchronize on both sides of the timed region. The step time is the median
over the K steps of the slowest rank's step (min / mean / max reported too).

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_PEAK_FALLBACK = 6553.6  # GB/s
FP64_PEAK_MEASURED = 36.9   # TFLOP/s, tools/microbench/fp64_peaks.cu on this pool (DMMA == DFMA)
DEFAULT_CONFIG = "cfg4"


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


def cpu_identity() -> dict:
    """the host the CPU baseline ran on: model string, physical cores and
    logical CPUs (the reference's acceptance header records the same,
    proj/tests/acceptance.cpp:70-93)"""
    model, cores, sockets = None, set(), set()
    phys = core = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if ":" not in line:
                    if phys is not None or core is not None:
                        cores.add((phys, core))
                    phys = core = None
                    continue
                k, v = [x.strip() for x in line.split(":", 1)]
                if k == "model name" and model is None:
                    model = v
                elif k == "physical id":
                    phys = v
                    sockets.add(v)
                elif k == "core id":
                    core = v
        if phys is not None or core is not None:
            cores.add((phys, core))
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "physical_cores": len(cores) or None,
            "sockets": len(sockets) or None, "logical_cpus": os.cpu_count(),
            "usable_cpus": usable}


def mapped_repo_libs():
    """shared objects of this repo mapped into the current process"""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                p = line.split()[-1] if line.strip() else ""
                if p.endswith(".so") and p.startswith(ROOT):
                    out.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(out)


def _nvml_index(local: int):
    """NVML handle selector for CUDA device `local` (CUDA_VISIBLE_DEVICES aware)"""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [x.strip() for x in vis.split(",") if x.strip()]
        if local < len(ids):
            return ids[local]
    return str(local)


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every few ms
    during the timed region, through NVML (nvidia-smi as a fallback)"""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int, period_s: float = 0.004):
        self.gpu = gpu_index
        self.period = period_s
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self.stop_ev = threading.Event()
        self.thread = None
        self.proc = None
        self.lines = []

    def start(self):
        try:
            import pynvml as N

            N.nvmlInit()
            sel = _nvml_index(self.gpu)
            h = (N.nvmlDeviceGetHandleByUUID(sel) if sel.startswith(("GPU-", "MIG-"))
                 else N.nvmlDeviceGetHandleByIndex(int(sel)))
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons

            def loop():
                while not self.stop_ev.is_set():
                    try:
                        self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                        r = int(get_reasons(h))
                        for bit, name in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    self.stop_ev.wait(self.period)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            self.kind = "nvml"
            return
        except Exception:
            pass
        self.kind = "nvidia-smi"
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={_nvml_index(self.gpu)}", f"--query-gpu={fields}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(
                target=lambda: [self.lines.append(l.strip()) for l in self.proc.stdout],
                daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def stop(self):
        self.stop_ev.set()
        if self.proc is not None:
            time.sleep(0.03)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    self.sm.append(float(parts[0]))
                    self.max_mhz = float(parts[1])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[2:6]):
                    if v.lower().startswith("active"):
                        self.reasons.add(nm)
        if self.thread:
            self.thread.join(timeout=2)
        if not self.sm:
            return None
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                "sm_mhz_min": min(self.sm), "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": getattr(self, "kind", None)}


# ---------------------------------------------------------------- processes
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("LRB_BENCH_SHARE_GPU") == "1":
        # functional test of the multi-rank path on fewer GPUs than ranks: the
        # ranks share devices (they never wait on one another's kernels: the
        # only collectives are host-side). The numbers are NOT a measurement;
        # the line is tagged.
        local = local % max(1, visible_gpus())
        print("bench.py: LRB_BENCH_SHARE_GPU=1, ranks share GPUs: a functional test, not a "
              "measurement", file=sys.stderr)
    pg = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # the only collectives are barriers and gathers of host scalars: gloo
        # keeps torch off the GPU entirely
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


def all_gather(pg, obj):
    if pg is None:
        return [obj]
    out = [None] * pg.get_world_size()
    pg.all_gather_object(out, obj)
    return out


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def visible_gpus() -> int:
    from paper_2311_07602_b200 import device_count

    return device_count()


def spawn_ranks(n: int) -> int:
    """run this script as n ranks (one process per GPU), wait for all; the
    first failing rank's exit code is returned and the others are stopped"""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env))
    rc = 0
    while procs:
        for p in list(procs):
            code = p.poll()
            if code is None:
                continue
            procs.remove(p)
            if code != 0 and rc == 0:
                rc = code
                for q in procs:
                    q.terminate()
        time.sleep(0.05)
    return rc


# ----------------------------------------------------------- workload slice
def item_roofline_s(w, i, hbm_gbs=None, fp64_tf=None):
    """per-item roofline time max(flops / P_fp64, bytes / BW_hbm)"""
    if hbm_gbs is None:
        hbm_gbs, _, fp64_tf, _ = load_peaks()
    return max(w.item_flops(i) / (fp64_tf * 1e12), w.item_bytes(i) / (hbm_gbs * 1e9))


def shard_ranges(w, world):
    """[(first global item, count)] per rank and the scaling mode.

    cfg4 (variable sizes): one batch split at equal cumulative per-item
    roofline time (lrb_shard_plan with costs); cfg5: the
    whole-box batch split evenly (the reference's contiguous fan-out,
    bench.hpp:69-75); every other config keeps one BASELINE batch per GPU
    (weak scaling) indexed globally."""
    from paper_2311_07602_b200 import shard_plan, workloads as W

    if isinstance(w, W.Variable):
        hbm, _, fp64, _ = load_peaks()
        cost = [item_roofline_s(w, i, hbm, fp64) for i in range(w.batch)]
        b = shard_plan(w.batch, world, cost)
        return [(b[r], b[r + 1] - b[r]) for r in range(world)], "strong"
    if w.name == "cfg5":
        b = shard_plan(w.batch, world)
        return [(b[r], b[r + 1] - b[r]) for r in range(world)], "strong"
    return [(r * w.batch, w.batch) for r in range(world)], "weak"


def scaling_of(w) -> str:
    """the scaling mode shard_ranges applies (host-only, no library call)"""
    from paper_2311_07602_b200 import workloads as W

    return "strong" if isinstance(w, W.Variable) or getattr(w, "name", "") == "cfg5" else "weak"


def rank_items(w, world, rank):
    """(first global item, count, scaling) of this rank"""
    spans, scaling = shard_ranges(w, world)
    return spans[rank][0], spans[rank][1], scaling


def traffic_from_profiles(config_name: str, items=None):
    """DRAM read+write bytes of one launch of the config's kernel(s) from the
    committed ncu summary (profiles/traffic.json). Entries record the items
    they were captured on; a launch over a different item count is scaled
    linearly and says so."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except Exception:
        return None
    e = d.get(config_name)
    if not isinstance(e, dict):
        return None
    e = dict(e)
    cap = e.get("items")
    if items is not None and cap and int(cap) != int(items):
        e["dram_bytes_per_launch"] = e["dram_bytes_per_launch"] * float(items) / float(cap)
        e["scaled_from_items"] = cap
    elif items is not None and not cap:
        return None  # capture size unknown: do not pair bytes of another launch size
    return e


# ------------------------------------------------------------- CPU baseline
def cpu_sample_run(w, items, threads):
    """time the reference binary (oracle/_ref, else the C restatement) on a
    bounded sample of the workload's items; returns (seconds, flops, bytes, kind)"""
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


def cpu_baseline(w, threads, target_s, what=None):
    items = pick_sample(w, threads, target_s)
    cpu_sample_run(w, items, threads)  # one untimed pass: threads, pages and clocks warm
    dt, fl, _, kind = cpu_sample_run(w, items, threads)
    d = {"value": round(fl / dt / 1e9, 3), "unit": "GFLOP/s", "cores": threads, "kind": kind,
         "sample": f"{len(items)} of {w.batch} items of {w.name} ({dt:.1f} s, after one untimed "
                   f"pass), per-item rate; "
                   f"std::thread contiguous split like naive_multiply_batch"}
    d.update(cpu_identity())
    return d


def run_reference_arm(args, w, world, rank):
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    ident = cpu_identity()
    threads = ident["usable_cpus"] or 1
    # each step a bounded sample, sized so the W + K steps end within minutes
    per_step_s = min(args.ref_seconds, 150.0 / max(1, args.steps + args.warmup))
    items = pick_sample(w, threads, per_step_s)
    for _ in range(max(0, args.warmup)):
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
    libs = mapped_repo_libs()
    if any("liblrb.so" in p for p in libs):
        raise RuntimeError(f"reference arm mapped the product library: {libs}")
    cb = {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": threads, "kind": kind,
          "sample": sample}
    cb.update(ident)
    line = {
        "metric": "batched FP64 GFLOP/s", "value": round(gflops, 3), "unit": "GFLOP/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": scaling_of(w),
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (counter RNG, uniform[-1,1))",
        "config": dict(w.describe(), sample_items=len(items)),
        "step_ms": {"median": round(t * 1e3, 3), "min": round(min(times) * 1e3, 3),
                    "max": round(max(times) * 1e3, 3)},
        "hbm_gbs": None,
        "cpu_baseline": cb,
        "e2e": {"value": round(gflops, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "native_libs": libs,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ timing
def timed_steps(ctx, stream, step, steps, warmup, pg, local, graphs=1):
    """W warm-up steps, then K timed steps. The K steps are captured into ONE
    CUDA graph with an event record between consecutive steps (event-record
    nodes), so the steps run back to back with no host launch gap and each
    step's device time is still read from its own pair of events. Returns
    (total ms, [per-step ms], launches, clocks). `graphs` is kept for
    callers that rotate buffers (consecutive captures of `step` rotate)."""
    for _ in range(warmup):
        step()
    stream.synchronize()
    evs = [ctx.event() for _ in range(steps + 1)]
    with ctx.capture(stream) as cap:
        evs[0].record(stream)
        for i in range(steps):
            step()
            evs[i + 1].record(stream)
    graph = cap.graph
    sampler = ClockSampler(local)
    sampler.start()
    barrier(pg)
    stream.synchronize()
    launches0 = ctx.launch_count
    graph.launch(stream)
    stream.synchronize()
    barrier(pg)
    clocks = sampler.stop()
    per = [evs[i].elapsed_ms(evs[i + 1]) for i in range(steps)]
    return evs[0].elapsed_ms(evs[-1]), per, ctx.launch_count - launches0, clocks


def job_step_stats(pg, per_rank_steps, ms_total):
    """per step: the slowest rank's time; reported median / mean / min / max,
    plus each rank's total and median (the per-GPU spread)"""
    mine = {"steps": per_rank_steps, "total": ms_total}
    allr = all_gather(pg, mine)
    K = len(per_rank_steps)
    job = [max(r["steps"][i] for r in allr) for i in range(K)]
    med = statistics.median(job)
    ranks = [{"rank": i, "ms_total": round(r["total"], 4),
              "ms_median": round(statistics.median(r["steps"]), 4)} for i, r in enumerate(allr)]
    meds = [r["ms_median"] for r in ranks]
    stats = {"median": round(med, 4), "mean": round(statistics.mean(job), 4),
             "min": round(min(job), 4), "max": round(max(job), 4),
             "per_rank": ranks,
             "rank_spread": round((max(meds) - min(meds)) / max(meds), 4) if meds and max(meds) else 0.0}
    return med, stats


def roofline(flops, bytes_, ms, hbm_peak, fp64_peak, hbm_src, fp64_src):
    intensity = flops / bytes_
    fp64_bound = intensity * hbm_peak * 1e9 >= fp64_peak * 1e12
    if fp64_bound:
        ach = flops / (ms * 1e-3) / 1e12
        r = {"bound": "tensor", "achieved": round(ach, 3), "peak": fp64_peak, "unit": "TFLOP/s",
             "frac": round(ach / fp64_peak, 4),
             "peak_source": fp64_src + " (FP64 DMMA; MEASURED_PEAKS.json has no FP64 figure)"}
    else:
        ach = bytes_ / (ms * 1e-3) / 1e9
        r = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
             "frac": round(ach / hbm_peak, 4), "peak_source": hbm_src}
    r["roofline_frac"] = round(flops / (ms * 1e-3) /
                               min(fp64_peak * 1e12, intensity * hbm_peak * 1e9), 4)
    r["algorithmic"] = bytes_
    return r


# ------------------------------------------------------------------ GPU arm
def alloc_inputs(ctx, w, first, count):
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
    """cfg4 items [first, first + count) on one rank: three arenas with
    256-B aligned item bases, generated on device from global item indices,
    and the pointer-array plan over them"""

    def __init__(self, ctx, w, first, count):
        from paper_2311_07602_b200 import workloads as W

        self.items = list(range(first, first + count))
        self.offs, (na, nb, nc) = W.variable_layout(w, self.items)
        self.sizes = (na, nb, nc)
        self.arena = [ctx.malloc(na), ctx.malloc(nb), ctx.malloc(nc)]
        self.pa = [self.arena[0].ptr + o[0] for o in self.offs]
        self.pb = [self.arena[1].ptr + o[1] for o in self.offs]
        self.pc = [self.arena[2].ptr + o[2] for o in self.offs]
        self.bs = [w.bs[i] for i in self.items]
        self.rs = [w.rs[i] for i in self.items]
        ctx.fill_uniform_ptr(self.pa, self.bs, self.bs, self.bs, w.seed, W.ROLE_A, first)
        ctx.fill_uniform_ptr(self.pb, self.bs, self.rs, self.bs, w.seed, W.ROLE_B, first)
        self.plan = ctx.ptr_plan("C", "N", "N", self.bs, self.rs, self.bs, self.pa, self.bs,
                                 self.pb, self.bs, self.pc, self.bs, 0.0)
        ctx.synchronize()


def host_mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 16 << 30


def run_e2e_variable(args, ctx, w, vs, pg):
    """cfg4 through lrb_dgemm_ptr_batched_host: every item's A_i, B_i, C_i in
    pinned HOST arenas (the same 256-B aligned layout), H2D + kernels + D2H of
    the results inside the timed region"""
    na, nb, nc = vs.sizes
    budget = int(0.4 * host_mem_available())
    n = len(vs.items)
    if na + nb + nc > budget:  # the largest item prefix that fits the host
        acc = 0
        for i, o in enumerate(vs.offs):
            if o[0] + o[1] + o[2] > budget:
                n = i
                break
        na, nb, nc = vs.offs[n][0], vs.offs[n][1], vs.offs[n][2]
    hA, hB, hC = ctx.pinned(na // 8), ctx.pinned(nb // 8), ctx.pinned(nc // 8)
    from paper_2311_07602_b200.lrbatch import _check, lib

    _check(lib.lrb_memcpy_d2h(ctx._h, hA.ptr, vs.arena[0].ptr, na), ctx._h)
    _check(lib.lrb_memcpy_d2h(ctx._h, hB.ptr, vs.arena[1].ptr, nb), ctx._h)
    offs = vs.offs[:n]
    pa = [hA.ptr + o[0] for o in offs]
    pb = [hB.ptr + o[1] for o in offs]
    pc = [hC.ptr + o[2] for o in offs]
    bs, rs = vs.bs[:n], vs.rs[:n]

    def once():
        ctx.dgemm_ptr_batched_host("C", "N", "N", bs, rs, bs, pa, bs, pb, bs, pc, bs, 0.0)

    once()
    barrier(pg)
    times = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        once()
        times.append(time.perf_counter() - t0)
    dt = all_max(pg, statistics.median(times))
    ids = vs.items[:n]
    fl_all = all_sum(pg, w.flops(ids))
    h2d = sum(8 * (b * b + b * r) for b, r in zip(bs, rs))
    d2h = sum(8 * b * r for b, r in zip(bs, rs))
    return {"value": round(fl_all / dt / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "items_per_rank": n, "ms_per_step": round(dt * 1e3, 2),
            "path": "lrb_dgemm_ptr_batched_host (pinned host blocks; coalesced runs, "
                    "3-stream chunked H2D / pointer-array kernels / D2H)"}


def run_gpu_arm_variable(args, w, world, rank, local, pg, spans, scaling):
    from paper_2311_07602_b200 import Context

    hbm_peak, hbm_src, fp64_peak, fp64_src = load_peaks()
    ctx = Context(local)
    stream = ctx.stream()
    first, count = spans[rank]
    vs = VariableSlice(ctx, w, first, count)
    ms_rank, per, launches, clocks = timed_steps(ctx, stream, lambda: vs.plan.execute(stream),
                                                 args.steps, args.warmup, pg, local)
    ms_step, stats = job_step_stats(pg, per, ms_rank)
    fl = w.flops(vs.items)
    by = w.bytes(vs.items)
    fl_all = all_sum(pg, fl)
    by_all = all_sum(pg, by)
    gflops = fl_all / (ms_step * 1e-3) / 1e9
    my_med = statistics.median(per)
    roof = roofline(fl, by, my_med, hbm_peak, fp64_peak, hbm_src, fp64_src)
    # the per-item roofline: sum over items of max(flops/P, bytes/BW)
    t_item = sum(item_roofline_s(w, i, hbm_peak, fp64_peak) for i in vs.items)
    roof["per_item_roofline_frac"] = round(t_item / (my_med * 1e-3), 4)
    # DMMA works on 8-column fragments: r_i pads to a multiple of 8 on the
    # tensor pipe; the padded figure is the pipe's own utilisation
    fl_pad = sum(2.0 * w.bs[i] * w.bs[i] * ((w.rs[i] + 7) // 8 * 8) for i in vs.items)
    roof["padded_dmma_frac"] = round(fl_pad / (my_med * 1e-3) / (fp64_peak * 1e12), 4)
    roof["kernel"] = ("lrb_varn_kernel (single-launch pointer-array kernel)"
                      if vs.plan.launches == 1 else
                      "lrb_gemm_kernel (pointer-array plan, %d launches)" % vs.plan.launches)
    roof["kernel_ms"] = round(my_med, 4)
    tr = traffic_from_profiles(w.name, count)
    roof["traffic"] = tr.get("dram_bytes_per_launch") if isinstance(tr, dict) else None
    e2e = run_e2e_variable(args, ctx, w, vs, pg) if args.e2e_steps > 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(w, cpu_identity()["usable_cpus"] or 1, args.ref_seconds)
    if rank == 0:
        cfg = dict(w.describe())
        cfg.update({"parallelism": f"shard{world} (independent items, no collective)",
                    "shards": [list(s) for s in spans],
                    "shard_rule": "equal cumulative per-item roofline time (lrb_shard_plan)",
                    "launches_per_step": vs.plan.launches,
                    "timed_launch": "one CUDA graph of the K steps, an event record node between steps",
                    "l2": "inputs larger than L2 (no flush)"})
        line = {
            "metric": "batched FP64 GFLOP/s", "value": round(gflops, 2), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device counter RNG, uniform[-1,1), BASELINE seeds)",
            "config": cfg, "hbm_gbs": round(by_all / (ms_step * 1e-3) / 1e9, 1),
            "step_ms": stats, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks, "gpu_launches": int(launches),
        }
        if os.environ.get("LRB_BENCH_SHARE_GPU") == "1":
            line["shared_gpu_test"] = True
        print(json.dumps(line), flush=True)
    ctx.close()


def run_gpu_arm(args, w, world, rank, local, pg):
    from paper_2311_07602_b200 import Context, select, workloads as W

    spans, scaling = shard_ranges(w, world)
    if isinstance(w, W.Variable):
        return run_gpu_arm_variable(args, w, world, rank, local, pg, spans, scaling)

    hbm_peak, hbm_src, fp64_peak, fp64_src = load_peaks()
    ctx = Context(local)
    stream = ctx.stream()
    first, count = spans[rank]

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

    if resident:
        def step():
            a, b, c = bufs[rot[0] % copies]
            rot[0] += 1
            gemm(ctx, w, a, b, c, count, stream)

        ms_rank, per, launches, clocks = timed_steps(ctx, stream, step, args.steps, args.warmup,
                                                     pg, local, graphs=copies)
    else:
        # chunked (cfg5 below 4 GPUs): each chunk regenerated untimed; a step's
        # time is the sum of its chunks' GEMM launches (events around each)
        e0, e1 = ctx.event(), ctx.event()

        def chunked_step():
            total = 0.0
            for c in range(nchunks):
                c0 = c * chunk
                cn = min(chunk, count - c0)
                ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, cn, w.seed, W.ROLE_A,
                                 first + c0, stream)
                ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, cn, w.seed, W.ROLE_B,
                                 first + c0, stream)
                e0.record(stream)
                gemm(ctx, w, A, B, Cd, cn, stream)
                e1.record(stream)
                stream.synchronize()
                total += e0.elapsed_ms(e1)
            return total

        for _ in range(args.warmup):
            chunked_step()
        sampler = ClockSampler(local)
        sampler.start()
        barrier(pg)
        per = [chunked_step() for _ in range(args.steps)]
        barrier(pg)
        clocks = sampler.stop()
        ms_rank = sum(per)
        launches = args.steps * nchunks  # only GEMM launches count
    ms_step, stats = job_step_stats(pg, per, ms_rank)
    cold = cold_single_call(ctx, stream, w, bufs[0], count, args.steps) if copies > 1 else None
    items_all = all_sum(pg, float(count))
    flops_all = w.item_flops() * items_all
    bytes_all = w.item_bytes() * items_all
    gflops = flops_all / (ms_step * 1e-3) / 1e9
    gbs = bytes_all / (ms_step * 1e-3) / 1e9

    # ---- dominant kernel roofline (this rank, per launch, median step)
    launches_per_step = max(1, launches // max(1, args.steps))
    per_launch_ms = statistics.median(per) / launches_per_step
    launch_items = count / nchunks
    sel = select(w.order, w.opA, w.opB, w.m, w.n, w.k, chunk, ctx)
    roof = roofline(w.item_flops() * launch_items, w.item_bytes() * launch_items, per_launch_ms,
                    hbm_peak, fp64_peak, hbm_src, fp64_src)
    tr = traffic_from_profiles(w.name, int(round(launch_items)))
    roof["traffic"] = tr.get("dram_bytes_per_launch") if isinstance(tr, dict) else None
    roof["kernel"] = ("lrb_panel_kernel<p256>" if sel["name"] == "p256" else
                      f"lrb_gemm_kernel<{sel['name']}>")
    roof["kernel_ms"] = round(per_launch_ms, 4)
    roof["items_per_launch"] = launch_items

    # ---- e2e through the host-buffer C-ABI (pinned host memory, copies timed)
    del A, B, Cd, bufs
    e2e = run_e2e(args, ctx, w, first, count, pg) if args.e2e_steps > 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(w, cpu_identity()["usable_cpus"] or 1, args.ref_seconds)

    if rank == 0:
        cfg = dict(w.describe())
        cfg.update({"items_per_rank": count, "global_items": int(items_all),
                    "shards": [list(s) for s in spans],
                    "timed_launch": ("one CUDA graph of the K steps, an event record node between "
                                     "steps") if resident else "eager launches",
                    "parallelism": f"shard{world} (independent items, no collective)",
                    "kernel_variant": sel["name"],
                    "l2": (f"{copies} rotating copies of inputs+outputs "
                           f"({per_item * count * copies / 2**20:.0f} MiB) > 3x L2"
                           if copies > 1 else "inputs larger than L2 (no flush)"),
                    "chunks_per_step": nchunks})
        if cold is not None:
            by = w.item_bytes() * count
            for k in ("evict", "flush"):
                cold[f"{k}_hbm_frac"] = round(by / (cold[f"{k}_ms"] * 1e-3) / 1e9 / hbm_peak, 4)
        line = {
            "metric": "batched FP64 GFLOP/s", "value": round(gflops, 2), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device counter RNG, uniform[-1,1), BASELINE seeds)",
            "config": cfg, "hbm_gbs": round(gbs, 1), "step_ms": stats, "cold_call": cold,
            "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": int(launches),
        }
        if os.environ.get("LRB_BENCH_SHARE_GPU") == "1":
            line["shared_gpu_test"] = True
        print(json.dumps(line), flush=True)
    ctx.close()


def cold_single_call(ctx, stream, w, buf, count, reps):
    """one launch at a time (outside the timed steps) with the working set
    out of L2: after a clean eviction (lrb_l2_evict: L2 refilled with clean
    lines) and after a memset flush (lrb_l2_flush: L2 full of dirty lines the
    kernel's reads must write back first); median ms of `reps` each"""
    A, B, Cd = buf
    e0, e1 = ctx.event(), ctx.event()
    out = {}
    for mode in ("evict", "flush"):
        ts = []
        for _ in range(max(3, reps)):
            (ctx.l2_evict if mode == "evict" else ctx.l2_flush)(stream)
            e0.record(stream)
            gemm(ctx, w, A, B, Cd, count, stream)
            e1.record(stream)
            stream.synchronize()
            ts.append(e0.elapsed_ms(e1))
        out[f"{mode}_ms"] = round(statistics.median(ts), 5)
    return out


def run_e2e(args, ctx, w, first, count, pg):
    """same metric through lrb_dgemm_strided_batched_host: pinned host inputs,
    H2D + kernels + D2H of the result inside the timed region"""
    # whole batch when it fits the host's pinned-memory budget (cfg5's 288 GiB
    # does not: its e2e runs on the largest prefix that does)
    per_item = 8 * (w.sA + w.sB + w.sC)
    budget = min(16 << 30, int(0.4 * host_mem_available()))
    n = min(count, args.e2e_items) if args.e2e_items else min(count, max(1, budget // per_item))
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
    times = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        once()
        times.append(time.perf_counter() - t0)
    dt = all_max(pg, statistics.median(times))
    items_all = all_sum(pg, float(n))
    return {"value": round(w.item_flops() * items_all / dt / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(8 * (w.sA + w.sB) * n),
            "d2h_bytes_per_step": int(8 * w.sC * n), "items_per_rank": n,
            "ms_per_step": round(dt * 1e3, 2),
            "path": "lrb_dgemm_strided_batched_host (3-stream chunked H2D/kernel/D2H)"}


def run_plan_only(args, w, world, rank, pg):
    """each rank reports the item range the planner gives it; rank 0 prints
    the gathered plan (no GPU work)"""
    spans, scaling = shard_ranges(w, world)
    first, count = spans[rank]
    mine = {"rank": rank, "begin": first, "end": first + count, "items": count,
            "pid": os.getpid()}
    from paper_2311_07602_b200 import workloads as W

    if isinstance(w, W.Variable):
        hbm, _, fp64, _ = load_peaks()
        mine["roofline_s"] = sum(item_roofline_s(w, i, hbm, fp64)
                                 for i in range(first, first + count))
    allr = all_gather(pg, mine)
    if rank == 0:
        print(json.dumps({"plan_only": True, "n_gpus": world, "config": w.describe(),
                          "scaling": scaling, "ranks": allr}), flush=True)


def run_reference(args, w, world, rank):
    """the reference arm: the reference's own CPU implementation of the
    workload, rank 0 only; nothing from the product package is loaded"""
    if rank != 0:
        return
    from paper_2311_07602_b200 import workloads as W
    import bench_rows as R

    bench_mod = sys.modules[__name__]
    if isinstance(w, W.LowRank):
        R.run_lowrank_reference(args, w, world, rank, bench_mod)
    elif isinstance(w, W.Blr):
        R.run_blr_reference(args, w, world, rank, bench_mod)
    elif isinstance(w, (W.LrExpand, W.BlrDense)):
        R.run_expand_reference(args, w, world, rank, bench_mod)
    else:
        run_reference_arm(args, w, world, rank)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="lrb", choices=["lrb", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-items", type=int, default=0, help="0 = the rank's whole batch")
    ap.add_argument("--ref-seconds", type=float, default=4.0,
                    help="CPU work per reference-arm step / cpu_baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--plan-only", action="store_true",
                    help="print each rank's item range from the shard planner and exit")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.warmup < 3 and args.impl == "lrb" and not args.plan_only:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    from paper_2311_07602_b200 import workloads as W

    w = W.get(args.config)
    launched = "WORLD_SIZE" in os.environ
    if launched and int(os.environ["WORLD_SIZE"]) != args.gpus and args.gpus != 1:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}",
              file=sys.stderr)
        sys.exit(2)
    if not launched and args.gpus > 1:
        if args.impl == "reference":
            # rank 0 alone runs the CPU reference: no other process is needed
            run_reference(args, w, args.gpus, 0)
            return
        if not args.plan_only:
            have = visible_gpus()
            if have < args.gpus:
                print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
                      file=sys.stderr)
                sys.exit(2)
        sys.exit(spawn_ranks(args.gpus))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, w, world, rank)  # ranks > 0 exit without work
        return
    world, rank, local, pg = dist_setup()
    if args.plan_only:
        run_plan_only(args, w, world, rank, pg)
    else:
        import bench_rows as R

        bench_mod = sys.modules[__name__]
        if isinstance(w, W.LowRank):
            R.run_lowrank_gpu(args, w, world, rank, local, pg, bench_mod)
        elif isinstance(w, W.Blr):
            R.run_blr_gpu(args, w, world, rank, local, pg, bench_mod)
        elif isinstance(w, (W.LrExpand, W.BlrDense)):
            R.run_expand_gpu(args, w, world, rank, local, pg, bench_mod)
        else:
            run_gpu_arm(args, w, world, rank, local, pg)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    if __package__ is None and os.path.basename(sys.argv[0]) == "bench.py":
        sys.modules.setdefault("bench", sys.modules[__name__])
    main()
