#!/usr/bin/env python3
"""Minimal driver for ncu: generate one config's inputs on device and launch
the GEMM `--launches` times (no CPU work, no e2e).

    python tools/profile_one.py --config cfg2 [--variant sq] [--launches 2] [--items N]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2311_07602_b200 import Context, workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--items", type=int, default=0)
    args = ap.parse_args()
    ctx = Context(0)
    w = W.get(args.config)
    if isinstance(w, W.Variable):
        items = list(range(w.batch if not args.items else args.items))
        offs, (na, nb, nc) = W.variable_layout(w, items)
        arena = [ctx.malloc(na), ctx.malloc(nb), ctx.malloc(nc)]
        bs = [w.bs[i] for i in items]
        rs = [w.rs[i] for i in items]
        pa = [arena[0].ptr + o[0] for o in offs]
        pb = [arena[1].ptr + o[1] for o in offs]
        pc = [arena[2].ptr + o[2] for o in offs]
        ctx.fill_uniform_ptr(pa, bs, bs, bs, w.seed, W.ROLE_A)
        ctx.fill_uniform_ptr(pb, bs, rs, bs, w.seed, W.ROLE_B)
        plan = ctx.ptr_plan("C", "N", "N", bs, rs, bs, pa, bs, pb, bs, pc, bs, 0.0)
        for _ in range(args.launches):
            plan.execute()
        ctx.synchronize()
        return
    count = args.items or w.batch
    A, B, Cd = ctx.empty(w.sA * count), ctx.empty(w.sB * count), ctx.empty(w.sC * count)
    ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, count, w.seed, W.ROLE_A)
    ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, count, w.seed, W.ROLE_B)
    ctx.set_variant_override(args.variant)
    for _ in range(args.launches):
        ctx.dgemm_strided_batched(w.order, w.opA, w.opB, w.m, w.n, w.k, 0.0, A, w.lda, w.sA, B,
                                  w.ldb, w.sB, Cd, w.ldc, w.sC, count)
    ctx.synchronize()
    print(f"{args.config}: {args.launches} launches of {count} items ok")


if __name__ == "__main__":
    main()
