"""bench.py legs for the widened §8(f) rows, same contract as the GEMM legs.

  --config lr_r{R}_b{B}[_n{batch}]      the paper's batched low-rank product
                                        (lrb_lowrank_multiply; reference arm:
                                        the reference's naive_multiply_batch)
  --config blr_n{N}_b{B}_r{R}_k{nrhs}   BLR multi-RHS matvec (lrb_blr_matvec;
                                        reference arm: the reference's
                                        blr_matvec / blr_matvec_naive)

A step is one full product / matvec with inputs resident in HBM; the K timed
steps replay as one CUDA graph. GFLOP/s follows the reference's accounting
(4r^3 + 2r^2 b per low-rank item; 2mnk per product of the matvec).
"""
from __future__ import annotations

import json
import os
import statistics
import time

import numpy as np


def _roof(fl, by, ms, hbm, fp64, fsrc, hsrc, name=None):
    intensity = fl / by
    fp64_bound = intensity * hbm * 1e9 >= fp64 * 1e12
    if fp64_bound:
        ach = fl / (ms * 1e-3) / 1e12
        r = {"bound": "tensor", "achieved": round(ach, 3), "peak": fp64, "unit": "TFLOP/s",
             "frac": round(ach / fp64, 4), "peak_source": fsrc}
    else:
        ach = by / (ms * 1e-3) / 1e9
        r = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
             "frac": round(ach / hbm, 4), "peak_source": hsrc}
    r["roofline_frac"] = round(fl / (ms * 1e-3) / min(fp64 * 1e12, intensity * hbm * 1e9), 4)
    r["algorithmic"] = by
    r["traffic"] = None
    if name:
        from bench import traffic_from_profiles

        tr = traffic_from_profiles(name)
        if isinstance(tr, dict):
            # dram read + write of one step (summed over its launches), ncu --set full
            r["traffic"] = tr.get("dram_bytes_per_launch")
            r["traffic_launches"] = tr.get("launches")
    return r


def _timed(ctx, stream, step, steps, warmup, pg, B, local):
    """bench.timed_steps: the K steps as one CUDA graph, event nodes between steps;
    returns (median step ms of this rank, launches, clocks, job step stats)"""
    total, per, launches, clocks = B.timed_steps(ctx, stream, step, steps, warmup, pg, local)
    med, stats = B.job_step_stats(pg, per, total)
    return statistics.median(per), med, launches, clocks, stats


# ------------------------------------------------------------ low-rank product
def lowrank_inputs_host(w, items):
    from paper_2311_07602_b200 import lowrank as L

    b = L.LowRankBatch.random(items, w.block, w.rank, w.seed)
    return b


def run_lowrank_gpu(args, w, world, rank, local, pg, B):
    from paper_2311_07602_b200 import Context
    from paper_2311_07602_b200 import lowrank as L

    hbm, hsrc, fp64, fsrc = B.load_peaks()
    ctx = Context(local)
    s = ctx.stream()
    n, r, blk = w.batch, w.rank, w.block
    bufs = [ctx.empty(n * r * blk), ctx.empty(n * blk * r), ctx.empty(n * r * r),
            ctx.empty(n * r * r), ctx.empty(n * r * r)]
    # roles as column-major views of the row-major items; global item offset per rank
    first = rank * n
    ctx.fill_uniform(bufs[0], blk, r, blk, r * blk, n, w.seed, 0, first)
    ctx.fill_uniform(bufs[1], r, blk, r, blk * r, n, w.seed, 1, first)
    ctx.fill_uniform(bufs[2], r, r, r, r * r, n, w.seed, 2, first)
    ctx.fill_uniform(bufs[3], r, r, r, r * r, n, w.seed, 3, first)
    ctx.synchronize()
    step = lambda: L.lowrank_multiply_device(ctx, n, blk, r, *bufs, stream=s)  # noqa: E731
    ms_med, ms_step, launches, clocks, stats = _timed(ctx, s, step, args.steps, args.warmup, pg,
                                                      B, local)
    fl_all, by_all = B.all_sum(pg, w.flops()), B.all_sum(pg, w.bytes())
    roof = _roof(w.flops(), w.bytes(), ms_med, hbm, fp64, fsrc, hsrc, w.name)
    per_step = launches // max(1, args.steps)
    roof["kernel"] = ("lrb_lowrank_kernel<R> (fused, one warp per item)" if r <= 32 else
                      f"lrb_lowrank_big_kernel<{r}> (one launch, T and E on chip)" if per_step == 1 else
                      "lrb_gemm_kernel x3 (T and E in the workspace)")
    roof["kernel_ms"] = round(ms_med * args.steps / max(1, launches), 4)
    e2e = None
    if args.e2e_steps > 0:
        hb = lowrank_inputs_host(w, n)
        pins = [ctx.pinned(a.size) for a in (hb.a_vt_batch, hb.b_u_batch, hb.a_x_batch,
                                            hb.b_x_batch, hb.g_xy_batch)]
        for p, a in zip(pins, (hb.a_vt_batch, hb.b_u_batch, hb.a_x_batch, hb.b_x_batch)):
            p.array[:] = a
        from paper_2311_07602_b200.lrbatch import _check, lib

        def once():
            _check(lib.lrb_lowrank_multiply_host(ctx._h, n, blk, r, *[p.ptr for p in pins]),
                   ctx._h)

        once()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            once()
        dt = B.all_max(pg, (time.perf_counter() - t0) / args.e2e_steps)
        e2e = {"value": round(fl_all / dt / 1e9, 2), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(8 * (2 * r * blk + 2 * r * r) * n),
               "d2h_bytes_per_step": int(8 * r * r * n), "ms_per_step": round(dt * 1e3, 2),
               "path": "lrb_lowrank_multiply_host (chunked H2D/kernel/D2H)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = lowrank_cpu(w, os.cpu_count() or 1, args.ref_seconds)
        cpu.pop("seconds", None)
    if rank == 0:
        cfg = dict(w.describe())
        cfg.update({"parallelism": f"shard{world} (independent items, no collective)",
                    "timed_launch": "one CUDA graph of the K steps (event nodes between steps)",
                    "l2": "inputs larger than L2 (no flush)" if w.bytes() > 3 * 132644864
                          else "inputs within 3x L2"})
        print(json.dumps({
            "metric": "batched FP64 GFLOP/s", "value": round(fl_all / (ms_step * 1e-3) / 1e9, 2),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device counter RNG, uniform[-1,1))", "config": cfg,
            "hbm_gbs": round(by_all / (ms_step * 1e-3) / 1e9, 1), "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "step_ms": stats,
            "gpu_launches": int(launches)}),
            flush=True)
    ctx.close()


LOWRANK_DRIVERS = {0: "naive_multiply_batch", 2: "packed_multiply"}


def _fastest(candidates, run):
    """the candidate with the highest rate on a short probe (the reference
    arm reports the reference at its best)"""
    best, best_rate = candidates[0], -1.0
    for c in candidates:
        rate = run(c)
        if rate > best_rate:
            best, best_rate = c, rate
    return best


def lowrank_cpu(w, threads, target_s, which=None):
    """The reference's own CPU driver on a bounded sample, timed inside the
    reference call (oracle.ref_last_seconds: not the copy into LowRankBatch):
    the faster on this host of packed_multiply (kernels.hpp:243-349, the
    paper's optimised path, plan for oracle.DEFAULT_MACHINE) and
    naive_multiply_batch (bench.hpp:55-77)."""
    import oracle as O

    probe = lowrank_inputs_host(w, max(1, 4 * threads))
    args = (probe.a_vt_batch, probe.b_u_batch, probe.a_x_batch, probe.b_x_batch)
    if O.ref_available():
        kind = "reference"

        def rate(c):
            O.ref_lowrank(c, probe.batch_size, w.block, w.rank, *args, workers=threads)
            return probe.batch_size / max(O.ref_last_seconds(), 1e-9)

        which = _fastest((2, 0), rate) if which is None else which
        what = LOWRANK_DRIVERS[which]
        per_item = 1.0 / rate(which) * threads
    else:
        kind, what = "port", "naive restatement"
        t0 = time.perf_counter()
        O.lowrank(probe.batch_size, w.block, w.rank, *args, threads=threads, mode=O.REF_COMPILED)
        per_item = (time.perf_counter() - t0) / probe.batch_size * threads
    items = int(min(w.batch, max(threads, threads * target_s / max(per_item, 1e-9))))
    b = lowrank_inputs_host(w, items)
    args = (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)
    t0 = time.perf_counter()
    if kind == "reference":
        O.ref_lowrank(which, items, w.block, w.rank, *args, workers=threads)
        dt = O.ref_last_seconds()
    else:
        O.lowrank(items, w.block, w.rank, *args, threads=threads, mode=O.REF_COMPILED)
        dt = time.perf_counter() - t0
    plan = f", plan {O.DEFAULT_MACHINE}" if (kind == "reference" and which == 2) else ""
    return {"value": round(w.item_flops() * items / dt / 1e9, 3), "unit": "GFLOP/s",
            "cores": threads, "kind": kind, "seconds": dt, "driver": which,
            "sample": f"{items} of {w.batch} items ({dt:.1f} s, driver call only), {what}{plan}"
                      " (the faster of packed_multiply / naive_multiply_batch here)"}


def run_lowrank_reference(args, w, world, rank, B):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    driver = lowrank_cpu(w, threads, min(1.0, args.ref_seconds))["driver"]  # picks the driver
    for _ in range(max(0, args.warmup - 1)):  # the driver pick above is the first
        lowrank_cpu(w, threads, min(1.0, args.ref_seconds), driver)
    vals = [lowrank_cpu(w, threads, args.ref_seconds, driver) for _ in range(args.steps)]
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[0], value=v)
    ms = 1e3 * statistics.median(x.pop("seconds") for x in vals)
    cb.pop("seconds", None)
    print(json.dumps({
        "metric": "batched FP64 GFLOP/s", "value": v, "unit": "GFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (counter RNG, uniform[-1,1))", "config": w.describe(),
        "cpu_baseline": dict(cb, **B.cpu_identity()),
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "native_libs": B.mapped_repo_libs()}), flush=True)


# ------------------------------------------------------------------ BLR matvec
def blr_host(w):
    from paper_2311_07602_b200 import DenseBlock
    from paper_2311_07602_b200 import blr as BL
    from paper_2311_07602_b200 import lowrank as L

    m = BL.BlrMatrix.random(w.n, w.block, w.rank, w.seed)
    rhs = DenseBlock(w.n, w.nrhs, L._uniform_vec(w.seed * 7919 + 1, 0,
                                                 np.arange(w.n * w.nrhs, dtype=np.uint64)))
    return m, rhs


def run_blr_gpu(args, w, world, rank, local, pg, B):
    from paper_2311_07602_b200 import Context
    from paper_2311_07602_b200.lrbatch import _check, lib

    hbm, hsrc, fp64, fsrc = B.load_peaks()
    ctx = Context(local)
    s = ctx.stream()
    m, rhs = blr_host(w)
    h = m.device_handle(ctx)
    d_rhs, d_y = ctx.to_device(rhs.data), ctx.empty(w.n * w.nrhs)
    step = lambda: _check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, w.nrhs, d_y.ptr,  # noqa
                                                     s.handle), ctx._h)
    ms_med, ms_step, launches, clocks, stats = _timed(ctx, s, step, args.steps, args.warmup, pg,
                                                      B, local)
    fl_all, by_all = B.all_sum(pg, w.flops()), B.all_sum(pg, w.bytes())
    roof = _roof(w.flops(), w.bytes(), ms_med, hbm, fp64, fsrc, hsrc, w.name)
    per_step = launches // max(1, args.steps)
    # (an odd count runs the fused launch between two padding copies: also
    # three launches, told apart by the shapes the fused kernel serves)
    k2 = w.nrhs + 1
    padded = (per_step == 3 and w.nrhs % 2 == 1 and k2 <= 16 and w.tiles >= 2 and
              w.rank in (4, 8, 16, 32) and w.block % 32 == 0 and
              os.environ.get("LRB_BLR_FUSED", "1") != "0")
    roof["kernel"] = ("blr_fused_kernel (one persistent launch per matvec)" if per_step == 1 else
                      "blr_repitch_kernel, blr_fused_kernel on rhs / y padded to an even count, "
                      "blr_repitch_kernel" if padded else
                      "blr_repitch_kernel x2 around lrb_gemm_kernel x2 + blr_couple_warp_kernel "
                      "(odd count, padded to even)" if per_step == 5 and w.nrhs % 2 == 1 else
                      "lrb_gemm_kernel x2 + blr_couple_warp_kernel per matvec")
    roof["kernel_ms"] = round(ms_med * args.steps / max(1, launches), 4)
    e2e = None
    if args.e2e_steps > 0:
        y = np.zeros(w.n * w.nrhs)

        def once():
            _check(lib.lrb_blr_matvec(ctx._h, h, rhs.data.ctypes.data, w.nrhs, y.ctypes.data),
                   ctx._h)

        once()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            once()
        dt = B.all_max(pg, (time.perf_counter() - t0) / args.e2e_steps)
        e2e = {"value": round(fl_all / dt / 1e9, 2), "unit": "GFLOP/s",
               "h2d_bytes_per_step": 8 * w.n * w.nrhs, "d2h_bytes_per_step": 8 * w.n * w.nrhs,
               "ms_per_step": round(dt * 1e3, 3),
               "path": "lrb_blr_matvec (matrix resident on the device, rhs/y host)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = blr_cpu(w, m, rhs)
        cpu.pop("seconds", None)
    if rank == 0:
        cfg = dict(w.describe())
        cfg.update({"parallelism": f"replicas{world} (one matvec per GPU, no collective)",
                    "timed_launch": "one CUDA graph of the K steps (event nodes between steps)",
                    "l2": (f"matrix streamed once per step, {w.bytes() / 132644864:.1f}x the L2 "
                           "(no flush)")})
        print(json.dumps({
            "metric": "batched FP64 GFLOP/s", "value": round(fl_all / (ms_step * 1e-3) / 1e9, 2),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter RNG, uniform[-1,1))", "config": cfg,
            "hbm_gbs": round(by_all / (ms_step * 1e-3) / 1e9, 1), "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "step_ms": stats,
            "gpu_launches": int(launches)}),
            flush=True)
    ctx.close()


def blr_cpu(w, m, rhs, which=None):
    """The reference's BLR matvec on the host, timed inside the reference
    call (not building its BlrMatrix): the faster here of blr_matvec
    (blr.hpp:141-175, packed per tile row, all workers, plan for
    oracle.DEFAULT_MACHINE) and blr_matvec_naive (blr.hpp:179-202)."""
    import oracle as O

    diag, u, x, vt = m.packed_arrays()
    threads = os.cpu_count() or 1
    if O.ref_available():
        kind = "reference"

        def run(c):
            O.ref_blr_matvec(c, w.n, w.block, w.rank, diag, u, x, vt, rhs.data, w.nrhs,
                             workers=threads)
            return O.ref_last_seconds()

        which = _fastest((0, 1), lambda c: 1.0 / max(run(c), 1e-9)) if which is None else which
        dt = run(which)
        what = (f"blr_matvec (packed, plan {O.DEFAULT_MACHINE}, {threads} workers)" if which == 0
                else "blr_matvec_naive (single thread)")
    else:
        t0 = time.perf_counter()
        O.blr_matvec(w.n, w.block, w.rank, diag, u, x, vt, rhs.data, w.nrhs, mode=O.REF_COMPILED)
        kind, what = "port", "blr_matvec_naive restatement"
        dt = time.perf_counter() - t0
    return {"value": round(w.flops() / dt / 1e9, 3), "unit": "GFLOP/s",
            "cores": threads if (kind == "reference" and which == 0) else 1, "kind": kind,
            "seconds": dt, "driver": which,
            "sample": f"one full matvec ({dt:.3f} s, driver call only): {what}"}


def run_blr_reference(args, w, world, rank, B):
    if rank != 0:
        return
    m, rhs = blr_host(w)
    driver = blr_cpu(w, m, rhs)["driver"]  # picks the driver
    for _ in range(max(0, args.warmup - 1)):  # the driver pick above is the first
        blr_cpu(w, m, rhs, driver)
    vals = [blr_cpu(w, m, rhs, driver) for _ in range(args.steps)]
    v = statistics.median(x["value"] for x in vals)
    ms = 1e3 * statistics.median(x.pop("seconds") for x in vals)
    print(json.dumps({
        "metric": "batched FP64 GFLOP/s", "value": v, "unit": "GFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter RNG, uniform[-1,1))", "config": w.describe(),
        "cpu_baseline": dict(vals[0], value=v, **B.cpu_identity()),
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "native_libs": B.mapped_repo_libs()}), flush=True)


# ------------------------------------------- low-rank expansion / BLR dense
def _expand_host(w, items, first=0):
    """seeded U, X, Vt host arrays for items [first, first+items) (counter RNG)"""
    from paper_2311_07602_b200 import lowrank as L
    from paper_2311_07602_b200 import workloads as W

    m, r = w.m, w.rank
    out = []
    for role, per in ((0, m * r), (1, r * r), (2, r * m)):
        key = W.stream_key(w.seed, role)
        idx = np.arange(per, dtype=np.uint64)
        out.append(np.concatenate([L._uniform_vec(key, first + it, idx) for it in range(items)]))
    return out


def expand_cpu(w, threads, target_s):
    """the reference's expansion on the host: (U X) Vt per item through its
    gemm_naive_raw (dense_gemm_naive's arithmetic), items split over all
    threads; or reconstruct_dense itself (single-threaded, as the reference
    has it). Timed inside the reference call."""
    import oracle as O
    from paper_2311_07602_b200 import blr as BL
    from paper_2311_07602_b200 import workloads as W

    if isinstance(w, W.BlrDense):
        m = BL.BlrMatrix.random(w.n, w.block, w.rank, w.seed)
        args = (w.n, w.block, w.rank) + m.packed_arrays()
        if O.ref_available():
            O.ref_blr_reconstruct(*args)
            dt, kind = O.ref_last_seconds(), "reference"
        else:
            t0 = time.perf_counter()
            O.blr_reconstruct(*args, mode=O.REF_COMPILED)
            dt, kind = time.perf_counter() - t0, "port"
        return {"value": round(w.flops() / dt / 1e9, 3), "unit": "GFLOP/s", "cores": 1,
                "kind": kind, "seconds": dt,
                "sample": f"one full reconstruct_dense ({dt:.2f} s, single-threaded as in the"
                          " reference)"}
    probe = max(threads, 2 * threads)
    u, x, vt = _expand_host(w, probe)
    if not O.ref_available():
        t0 = time.perf_counter()
        O.lowrank_expand(probe, w.m, w.m, w.rank, u, x, vt, mode=O.REF_COMPILED)
        per_item = (time.perf_counter() - t0) / probe * threads
        kind = "port"
    else:
        O.ref_lowrank_expand(probe, w.m, w.m, w.rank, u, x, vt, workers=threads)
        per_item = O.ref_last_seconds() / probe * threads
        kind = "reference"
    items = int(min(w.batch, max(threads, threads * target_s / max(per_item, 1e-9))))
    u, x, vt = _expand_host(w, items)
    t0 = time.perf_counter()
    if kind == "reference":
        O.ref_lowrank_expand(items, w.m, w.m, w.rank, u, x, vt, workers=threads)
        dt = O.ref_last_seconds()
    else:
        O.lowrank_expand(items, w.m, w.m, w.rank, u, x, vt, mode=O.REF_COMPILED)
        dt = time.perf_counter() - t0
    return {"value": round(w.item_flops() * items / dt / 1e9, 3), "unit": "GFLOP/s",
            "cores": threads if kind == "reference" else 1, "kind": kind, "seconds": dt,
            "sample": f"{items} of {w.batch} items ({dt:.1f} s, products only): (U X) Vt via"
                      " the reference's gemm_naive_raw, contiguous split over threads"}


def run_expand_gpu(args, w, world, rank, local, pg, B):
    from paper_2311_07602_b200 import Context
    from paper_2311_07602_b200 import blr as BL
    from paper_2311_07602_b200 import workloads as W

    hbm, hsrc, fp64, fsrc = B.load_peaks()
    ctx = Context(local)
    s = ctx.stream()
    dense = isinstance(w, W.BlrDense)
    if dense:
        mat = BL.BlrMatrix.random(w.n, w.block, w.rank, w.seed)
        mat.device_handle(ctx)
        out = ctx.empty(w.n * w.n)
        step = lambda: mat.reconstruct_dense_device(ctx, out, stream=s)  # noqa: E731
        fl, by = w.flops(), w.bytes()
        kernel = "dense"
    else:
        m, r, n = w.m, w.rank, w.batch
        bufs = [ctx.empty(n * m * r), ctx.empty(n * r * r), ctx.empty(n * r * m)]
        first = rank * n
        ctx.fill_uniform(bufs[0], r, m, r, m * r, n, w.seed, 0, first)
        ctx.fill_uniform(bufs[1], r, r, r, r * r, n, w.seed, 1, first)
        ctx.fill_uniform(bufs[2], m, r, m, r * m, n, w.seed, 2, first)
        out = ctx.empty(n * m * m)
        ctx.synchronize()
        step = lambda: BL.lowrank_expand_device(ctx, n, m, m, r, *bufs, out, stream=s)  # noqa
        fl, by = w.flops(), w.bytes()
        kernel = None  # named after a step: the kernel that served (UX) Vt
    ms_med, ms_step, launches, clocks, stats = _timed(ctx, s, step, args.steps, args.warmup, pg,
                                                      B, local)
    fl_all, by_all = B.all_sum(pg, fl), B.all_sum(pg, by)
    roof = _roof(fl, by, ms_med, hbm, fp64, fsrc, hsrc, w.name)
    per_step = launches // max(1, args.steps)
    if kernel == "dense":
        kernel = ("blr_diag_kernel beside blr_recon_kernel (streaming (U X) Vt, TMA stores)"
                  if per_step == 2 else
                  "blr_diag_kernel + blr_ux_mma_kernel + lrb_gemm_kernel<q64, BlrTileProblem>")
    elif per_step == 1:
        kernel = "blr_recon_kernel (streaming (U X) Vt, UX on chip, TMA stores)"
    else:
        v = ctx.last_variant
        kernel = ("lrb_gemm_kernel<q64> (UX), then " +
                  ("lrb_panel_kernel<p256>" if v == "p256" else f"lrb_gemm_kernel<{v}>") +
                  " ((UX) Vt)")
    roof["kernel"] = kernel
    roof["kernel_ms"] = round(ms_med * args.steps / max(1, launches), 4)
    e2e = None
    if args.e2e_steps > 0:
        from paper_2311_07602_b200.lrbatch import _check, lib

        if dense:
            host = np.zeros(w.n * w.n)
            h = mat.device_handle(ctx)

            def once():
                _check(lib.lrb_blr_reconstruct_dense(ctx._h, h, host.ctypes.data, 0, None),
                       ctx._h)

            hb, ob = 0, 8 * w.n * w.n
            path = "lrb_blr_reconstruct_dense (host out; matrix resident on the device)"
            ratio = 1.0
        else:
            items = min(w.batch, args.e2e_items or 1024)
            hu, hx, hvt = _expand_host(w, items, rank * w.batch)
            pins = [ctx.pinned(a.size) for a in (hu, hx, hvt)] + [ctx.pinned(items * w.m * w.m)]
            for p_, a in zip(pins, (hu, hx, hvt)):
                p_.array[:] = a
            dbu = [ctx.empty(a.size) for a in (hu, hx, hvt)]
            dout = ctx.empty(items * w.m * w.m)
            e2s = ctx.stream()

            def once():
                for p_, d in zip(pins, dbu):  # synchronous copies from pinned memory
                    _check(lib.lrb_memcpy_h2d(ctx._h, d.ptr, p_.ptr, p_.nbytes), ctx._h)
                BL.lowrank_expand_device(ctx, items, w.m, w.m, w.rank, *dbu, dout, stream=e2s)
                e2s.synchronize()
                _check(lib.lrb_memcpy_d2h(ctx._h, pins[3].ptr, dout.ptr, pins[3].nbytes), ctx._h)

            hb = 8 * (hu.size + hx.size + hvt.size)
            ob = 8 * items * w.m * w.m
            path = f"H2D (pinned) + lrb_lowrank_expand + D2H, {items} items per step"
            ratio = items / w.batch
        once()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            once()
        dt = B.all_max(pg, (time.perf_counter() - t0) / args.e2e_steps)
        e2e = {"value": round(fl_all * ratio / dt / 1e9, 2), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(hb), "d2h_bytes_per_step": int(ob),
               "ms_per_step": round(dt * 1e3, 3), "path": path}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = expand_cpu(w, os.cpu_count() or 1, args.ref_seconds)
        cpu.pop("seconds", None)
    if rank == 0:
        cfg = dict(w.describe())
        cfg.update({"parallelism": (f"replicas{world}" if dense else f"shard{world}")
                    + " (no collective)", "timed_launch": "one CUDA graph of the K steps (event nodes between steps)",
                    "l2": "output larger than L2 (no flush)"})
        print(json.dumps({
            "metric": "batched FP64 GFLOP/s", "value": round(fl_all / (ms_step * 1e-3) / 1e9, 2),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter RNG, uniform[-1,1))", "config": cfg,
            "hbm_gbs": round(by_all / (ms_step * 1e-3) / 1e9, 1), "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "step_ms": stats,
            "gpu_launches": int(launches)}),
            flush=True)
    ctx.close()


def run_expand_reference(args, w, world, rank, B):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(max(0, args.warmup)):
        expand_cpu(w, threads, min(1.0, args.ref_seconds))
    vals = [expand_cpu(w, threads, args.ref_seconds) for _ in range(args.steps)]
    v = statistics.median(x["value"] for x in vals)
    ms = 1e3 * statistics.median(x.pop("seconds") for x in vals)
    print(json.dumps({
        "metric": "batched FP64 GFLOP/s", "value": v, "unit": "GFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter RNG, uniform[-1,1))", "config": w.describe(),
        "cpu_baseline": dict(vals[0], value=v, **B.cpu_identity()),
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "native_libs": B.mapped_repo_libs()}), flush=True)
