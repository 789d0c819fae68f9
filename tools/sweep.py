#!/usr/bin/env python3
"""Kernel-time sweep over every BASELINE config (1 GPU, inputs resident in HBM).

    python tools/sweep.py [--configs cfg1,cfg2,...] [--variants auto|n16,sq,...] [--reps 10]

Per config and variant: device ms per launch (CUDA events on the launching
stream, median of reps; L2 flushed between reps when the working set is
within 3x L2), GFLOP/s, algorithmic GB/s, and the fraction of the per-shape
roofline min(FP64 peak, I * HBM peak). One JSON line per measurement.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import load_peaks  # noqa: E402
from paper_2311_07602_b200 import Context, workloads as W  # noqa: E402

L2 = 132644864


def time_launches(ctx, stream, launch, reps, flush):
    e0, e1 = ctx.event(), ctx.event()
    for _ in range(3):
        launch()
    out = []
    for _ in range(reps):
        if flush:
            ctx.l2_evict(stream)  # clean eviction (no dirty write-backs in the timed launch)
        e0.record(stream)
        launch()
        e1.record(stream)
        stream.synchronize()
        out.append(e0.elapsed_ms(e1))
    return statistics.median(out), min(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(W.all_names()[:-1]))
    ap.add_argument("--variants", default="auto")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    hbm, _, fp64, _ = load_peaks()
    ctx = Context(0)
    stream = ctx.stream()
    for name in args.configs.split(","):
        w = W.get(name)
        if isinstance(w, W.Variable):
            items = list(range(w.batch))
            offs, (na, nb, nc) = W.variable_layout(w, items)
            arena = [ctx.malloc(na), ctx.malloc(nb), ctx.malloc(nc)]
            pa = [arena[0].ptr + o[0] for o in offs]
            pb = [arena[1].ptr + o[1] for o in offs]
            pc = [arena[2].ptr + o[2] for o in offs]
            ctx.fill_uniform_ptr(pa, w.bs, w.bs, w.bs, w.seed, W.ROLE_A)
            ctx.fill_uniform_ptr(pb, w.bs, w.rs, w.bs, w.seed, W.ROLE_B)
            plan = ctx.ptr_plan("C", "N", "N", w.bs, w.rs, w.bs, pa, w.bs, pb, w.bs, pc, w.bs,
                                0.0)
            med, best = time_launches(ctx, stream, lambda: plan.execute(stream), args.reps, False)
            fl, by = w.flops(), w.bytes()
            roof = min(fp64 * 1e12, fl / by * hbm * 1e9)
            print(json.dumps({"config": name, "variant": "auto(ptr)", "launches": plan.launches,
                              "ms": round(med, 4), "gflops": round(fl / med / 1e6, 1),
                              "gbs": round(by / med / 1e6, 1), "intensity": round(fl / by, 2),
                              "roofline_frac": round(fl / (med * 1e-3) / roof, 4)}), flush=True)
            del plan, arena
            continue
        count = w.batch
        free, _ = ctx.mem_info()
        per = 8 * (w.sA + w.sB + w.sC)
        count = min(count, int((free - (4 << 30)) // per))
        A, B, Cd = ctx.empty(w.sA * count), ctx.empty(w.sB * count), ctx.empty(w.sC * count)
        ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, count, w.seed, W.ROLE_A)
        ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, count, w.seed, W.ROLE_B)
        ctx.synchronize()
        variants = [None] if args.variants == "auto" else args.variants.split(",")
        for v in variants:
            ctx.set_variant_override(v)

            def launch():
                ctx.dgemm_strided_batched(w.order, w.opA, w.opB, w.m, w.n, w.k, 0.0, A, w.lda,
                                          w.sA, B, w.ldb, w.sB, Cd, w.ldc, w.sC, count, stream)

            flush = per * count < 3 * L2
            med, best = time_launches(ctx, stream, launch, args.reps, flush)
            fl, by = w.item_flops() * count, w.item_bytes() * count
            intensity = fl / by
            roof = min(fp64 * 1e12, intensity * hbm * 1e9)
            from paper_2311_07602_b200 import select

            sel = select(w.order, w.opA, w.opB, w.m, w.n, w.k, count, ctx)
            print(json.dumps({"config": name, "variant": sel["name"], "items": count,
                              "ms": round(med, 4), "ms_best": round(best, 4),
                              "gflops": round(fl / med / 1e6, 1), "gbs": round(by / med / 1e6, 1),
                              "intensity": round(intensity, 2),
                              "bound": "fp64" if intensity * hbm * 1e9 >= fp64 * 1e12 else "hbm",
                              "roofline_frac": round(fl / (med * 1e-3) / roof, 4),
                              "l2_flush": flush}), flush=True)
        ctx.set_variant_override(None)
        del A, B, Cd


if __name__ == "__main__":
    main()
