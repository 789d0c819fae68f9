#!/usr/bin/env python3
"""cfg2 diagnostics: normal vs broadcast operands (strideA = strideB = 0, all
operand loads hit L2, only the C write stream reaches DRAM), per variant."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_07602_b200 import Context, workloads as W  # noqa: E402


def main():
    variants = sys.argv[1].split(",") if len(sys.argv) > 1 else ["n64"]
    ctx = Context(0)
    s = ctx.stream()
    w = W.get("cfg2")
    A, B, Cd = ctx.empty(w.sA * w.batch), ctx.empty(w.sB * w.batch), ctx.empty(w.sC * w.batch)
    ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, w.batch, w.seed, 0)
    ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, w.batch, w.seed, 1)
    e0, e1 = ctx.event(), ctx.event()
    for v in variants:
        ctx.set_variant_override(v)
        for mode, sa, sb in (("normal", w.sA, w.sB), ("broadcast", 0, 0)):
            def go():
                ctx.dgemm_strided_batched("C", "N", "T", 512, 512, 32, 0.0, A, 512, sa, B, 512, sb,
                                          Cd, 512, w.sC, w.batch, s)
            for _ in range(3):
                go()
            ts = []
            for _ in range(7):
                e0.record(s)
                go()
                e1.record(s)
                s.synchronize()
                ts.append(e0.elapsed_ms(e1))
            ms = statistics.median(ts)
            print(json.dumps({"variant": v, "mode": mode, "ms": round(ms, 4),
                              "tflops": round(w.flops() / ms / 1e9, 2),
                              "frac_fp64": round(w.flops() / ms / 1e9 / 36.9, 4)}), flush=True)


if __name__ == "__main__":
    main()
