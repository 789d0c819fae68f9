#!/usr/bin/env python3
"""cfg2-class diagnostics: time one config per (variant, LRB_DEBUG_FLAGS)
combination, each in a fresh process so the env-read flags apply.

    python tools/probe_policy.py cfg2 q64,t64,sq 0,32,128
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, statistics, sys
sys.path.insert(0, %r)
from paper_2311_07602_b200 import Context, workloads as W
ctx = Context(0); s = ctx.stream(); w = W.get(%r)
A, B, Cd = ctx.empty(w.sA * w.batch), ctx.empty(w.sB * w.batch), ctx.empty(w.sC * w.batch)
ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, w.batch, w.seed, W.ROLE_A)
ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, w.batch, w.seed, W.ROLE_B)
ctx.set_variant_override(%r)
e0, e1 = ctx.event(), ctx.event()
def go():
    ctx.dgemm_strided_batched(w.order, w.opA, w.opB, w.m, w.n, w.k, 0.0, A, w.lda, w.sA, B, w.ldb,
                              w.sB, Cd, w.ldc, w.sC, w.batch, s)
for _ in range(3): go()
ts = []
for _ in range(9):
    e0.record(s); go(); e1.record(s); s.synchronize(); ts.append(e0.elapsed_ms(e1))
ms = statistics.median(ts)
print(json.dumps({"ms": round(ms, 4), "tflops": round(w.flops() / ms / 1e9, 2),
                  "frac_fp64": round(w.flops() / ms / 1e9 / 36.9, 4)}))
"""


def main():
    cfg = sys.argv[1]
    variants = sys.argv[2].split(",")
    flags = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0"]
    for v in variants:
        for f in flags:
            env = dict(os.environ, LRB_DEBUG_FLAGS=f)
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, v)], env=env,
                                 capture_output=True, text=True)
            rec = {"config": cfg, "variant": v, "flags": int(f)}
            try:
                rec.update(json.loads(out.stdout.strip().splitlines()[-1]))
            except Exception:
                rec["error"] = (out.stderr or out.stdout)[-300:]
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
