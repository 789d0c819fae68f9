#!/usr/bin/env python3
"""Time one strided GEMM shape per forced variant (device-resident, CUDA
events, median of reps).

    python tools/probe_shape.py R N N 256 16 1264 64 m16k64,m16t,m16
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_07602_b200 import Context  # noqa: E402


def main():
    order, opA, opB = sys.argv[1:4]
    m, n, k, batch = (int(x) for x in sys.argv[4:8])
    variants = sys.argv[8].split(",") if len(sys.argv) > 8 else [None]
    ctx = Context(0)
    s = ctx.stream()
    ra, ca = (k, m) if opA == "T" else (m, k)
    rb, cb = (n, k) if opB == "T" else (k, n)
    lda = ca if order == "R" else ra
    ldb = cb if order == "R" else rb
    ldc = n if order == "R" else m
    sA, sB, sC = ra * ca, rb * cb, m * n
    A, B, Cd = ctx.empty(sA * batch), ctx.empty(sB * batch), ctx.empty(sC * batch)
    A.fill_bytes(0)
    B.fill_bytes(0)
    e0, e1 = ctx.event(), ctx.event()
    for v in variants:
        ctx.set_variant_override(None if v in (None, "auto") else v)

        def go():
            ctx.dgemm_strided_batched(order, opA, opB, m, n, k, 0.0, A, lda, sA, B, ldb, sB, Cd,
                                      ldc, sC, batch, s)
        for _ in range(3):
            go()
        ts = []
        for _ in range(15):
            e0.record(s)
            go()
            e1.record(s)
            s.synchronize()
            ts.append(e0.elapsed_ms(e1))
        ms = statistics.median(ts)
        by = 8.0 * (sA + sB + sC) * batch
        print(json.dumps({"shape": [order, opA, opB, m, n, k, batch], "variant": v,
                          "used": ctx.last_variant, "us": round(ms * 1e3, 2),
                          "gbs": round(by / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
