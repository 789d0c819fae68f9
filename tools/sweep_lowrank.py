#!/usr/bin/env python3
"""Kernel-time sweep of the paper's batched low-rank product on one B200.

    python tools/sweep_lowrank.py [--ranks 8,16,32,64,128] [--blocks 512,1024,2048] [--batch 20000]

GFLOP/s uses the reference's accounting 4r^3 + 2r^2 b (low_rank.hpp:66-68);
algorithmic bytes 8(2rb + 3r^2) per item; roofline min(FP64, I * HBM).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import load_peaks  # noqa: E402
from paper_2311_07602_b200 import Context  # noqa: E402
from paper_2311_07602_b200 import lowrank as L  # noqa: E402
from paper_2311_07602_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="8,16,32,64,96,128")
    ap.add_argument("--blocks", default="512,1024,2048")
    ap.add_argument("--batch", type=int, default=20000)
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    hbm, _, fp64, _ = load_peaks()
    ctx = Context(0)
    s = ctx.stream()
    e0, e1 = ctx.event(), ctx.event()
    for r in map(int, args.ranks.split(",")):
        for b in map(int, args.blocks.split(",")):
            w = W.LowRank(f"lr_r{r}_b{b}", args.batch, b, r)
            n = w.batch
            bufs = [ctx.empty(n * r * b), ctx.empty(n * b * r), ctx.empty(n * r * r),
                    ctx.empty(n * r * r), ctx.empty(n * r * r)]
            # roles as column-major views of the row-major items (values only)
            ctx.fill_uniform(bufs[0], b, r, b, r * b, n, w.seed, 0)
            ctx.fill_uniform(bufs[1], r, b, r, b * r, n, w.seed, 1)
            ctx.fill_uniform(bufs[2], r, r, r, r * r, n, w.seed, 2)
            ctx.fill_uniform(bufs[3], r, r, r, r * r, n, w.seed, 3)
            go = lambda: L.lowrank_multiply_device(ctx, n, b, r, *bufs, stream=s)  # noqa: E731
            n0 = ctx.launch_count
            for _ in range(3):
                go()
            per_call = (ctx.launch_count - n0) // 3
            ts = []
            for _ in range(args.reps):
                e0.record(s)
                go()
                e1.record(s)
                s.synchronize()
                ts.append(e0.elapsed_ms(e1))
            ms = statistics.median(ts)
            fl, by = w.flops(), w.bytes()
            roof = min(fp64 * 1e12, fl / by * hbm * 1e9)
            print(json.dumps({"config": w.name, "batch": n, "ms": round(ms, 4),
                              "gflops": round(fl / ms / 1e6, 1), "gbs": round(by / ms / 1e6, 1),
                              "intensity": round(fl / by, 2),
                              "roofline_frac": round(fl / (ms * 1e-3) / roof, 4),
                              "path": ("fused TMA+DMMA (one warp per item)" if r <= 32 else
                                       "one launch, T and E on chip" if per_call == 1 else
                                       "3 batched GEMMs")}),
                  flush=True)
            del bufs


if __name__ == "__main__":
    main()
