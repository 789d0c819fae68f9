#!/usr/bin/env python3
"""A/B probe of the cfg4 pointer-array paths on one box: the single-launch
kernel under its tile orders, against the per-variant buckets.

    python tools/probe_varn.py [--reps 10] [--items N]
prints one JSON line per setting (median ms per execute, fraction of FP64 peak)
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2311_07602_b200 import Context, workloads as W  # noqa: E402

SETTINGS = [
    ("varn interleaved", {}),
    ("varn claim-ahead", {"LRB_DEBUG_FLAGS": "8"}),
    ("varn interleaved again", {}),
    ("varn claim-ahead again", {"LRB_DEBUG_FLAGS": "8"}),
    ("varn longest-first", {"LRB_VARN_ORDER": "1"}),
    ("varn item order", {"LRB_VARN_ORDER": "2"}),
    ("varn device-path order", {"LRB_VARN_ORDER": "3"}),
    ("varn no stores", {"LRB_DEBUG_FLAGS": "2"}),
    ("buckets", {"LRB_PTR_BUCKETS": "1"}),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--items", type=int, default=0)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    ctx = Context(0)
    w = W.get("cfg4")
    n = args.items or w.batch
    vs = bench.VariableSlice(ctx, w, 0, n)
    fl = w.flops(vs.items)
    s = ctx.stream()
    for dev_env in ({}, {"LRB_DEBUG_FLAGS": "16"}, {}, {"LRB_DEBUG_FLAGS": "16"}):
        if args.only and "device" not in args.only:
            break
        os.environ.pop("LRB_DEBUG_FLAGS", None)
        os.environ.update(dev_env)
        import numpy as np

        d = {kk: ctx.to_device(np.asarray(v, dtype=np.int64)) for kk, v in
             dict(m=vs.bs, n=vs.rs, k=vs.bs, lda=vs.bs, ldb=vs.bs, ldc=vs.bs, A=vs.pa, B=vs.pb,
                  C=vs.pc).items()}

        def dev_call():
            ctx.dgemm_ptr_batched_device("C", "N", "N", n, d["m"], d["n"], d["k"], d["A"],
                                         d["lda"], d["B"], d["ldb"], d["C"], d["ldc"], 0.0,
                                         None, s)

        for _ in range(3):
            dev_call()
        s.synchronize()
        ts = []
        for _ in range(args.reps):
            e0, e1 = ctx.event(), ctx.event()
            e0.record(s)
            dev_call()
            e1.record(s)
            s.synchronize()
            ts.append(e0.elapsed_ms(e1))
        ms = statistics.median(ts)
        print(json.dumps({"setting": "device descriptors (lrb_dgemm_ptr_batched_device)",
                          "env": dev_env,
                          "items": n, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 2),
                          "frac": round(fl / ms / 1e9 / 36.9, 4)}), flush=True)
    for name, env in SETTINGS:
        if args.only and args.only not in name:
            continue
        for k in ("LRB_VARN_ORDER", "LRB_DEBUG_FLAGS", "LRB_PTR_BUCKETS"):
            os.environ.pop(k, None)
        os.environ.update(env)
        plan = ctx.ptr_plan("C", "N", "N", vs.bs, vs.rs, vs.bs, vs.pa, vs.bs, vs.pb, vs.bs,
                            vs.pc, vs.bs, 0.0)
        for _ in range(3):
            plan.execute(s)
        s.synchronize()
        ts = []
        for _ in range(args.reps):
            e0, e1 = ctx.event(), ctx.event()
            e0.record(s)
            plan.execute(s)
            e1.record(s)
            s.synchronize()
            ts.append(e0.elapsed_ms(e1))
        ms = statistics.median(ts)
        print(json.dumps({"setting": name, "env": env, "items": n, "launches": plan.launches,
                          "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 2),
                          "frac": round(fl / ms / 1e9 / 36.9, 4)}), flush=True)
        plan.destroy()


if __name__ == "__main__":
    main()
