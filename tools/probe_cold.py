#!/usr/bin/env python3
"""cfg1 (256 x 256x256 . 256x16) as a single cold launch: per tile variant and
per L2 state before the launch (memset flush = dirty lines written back during
the kernel, clean eviction, warm), plus the launch floor (one tiny item).

    python tools/probe_cold.py [--reps 20] [--variants n16t,n16,n16h]
one JSON line per setting: median / min ms, fraction of the HBM roofline
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--variants", default="auto,n16t,n16,n16h,n8")
    ap.add_argument("--config", default="cfg1")
    args = ap.parse_args()
    hbm, _, _, _ = load_peaks()
    ctx = Context(0)
    s = ctx.stream()
    w = W.get(args.config)
    A, B, Cd = ctx.empty(w.sA * w.batch), ctx.empty(w.sB * w.batch), ctx.empty(w.sC * w.batch)
    ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, w.batch, w.seed, W.ROLE_A)
    ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, w.batch, w.seed, W.ROLE_B)
    ctx.synchronize()
    by = w.item_bytes() * w.batch
    e0, e1 = ctx.event(), ctx.event()

    def run(batch):
        ctx.dgemm_strided_batched(w.order, w.opA, w.opB, w.m, w.n, w.k, 0.0, A, w.lda, w.sA, B,
                                  w.ldb, w.sB, Cd, w.ldc, w.sC, batch, s)

    for v in args.variants.split(","):
        ctx.set_variant_override(None if v == "auto" else v)
        for mode in ("flush", "evict", "warm"):
            ts = []
            for _ in range(3):
                run(w.batch)
            for _ in range(args.reps):
                if mode == "flush":
                    ctx.l2_flush(s)
                elif mode == "evict":
                    ctx.l2_evict(s)
                e0.record(s)
                run(w.batch)
                e1.record(s)
                s.synchronize()
                ts.append(e0.elapsed_ms(e1))
            ms = statistics.median(ts)
            print(json.dumps({"config": args.config, "variant": v, "ran": ctx.last_variant,
                              "l2_before": mode, "ms": round(ms, 5), "ms_min": round(min(ts), 5),
                              "gbs": round(by / ms / 1e6, 1),
                              "hbm_frac": round(by / ms / 1e6 / hbm, 4)}), flush=True)
    # the launch floor: one item of the same shape, after a clean eviction
    ctx.set_variant_override(None)
    ts = []
    for _ in range(args.reps):
        ctx.l2_evict(s)
        e0.record(s)
        run(1)
        e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_ms(e1))
    print(json.dumps({"config": args.config, "probe": "one item (launch floor)",
                      "ms": round(statistics.median(ts), 5)}), flush=True)


if __name__ == "__main__":
    main()
