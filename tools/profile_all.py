#!/usr/bin/env python3
"""One launch of the auto-selected kernel per BASELINE config, in a fixed
order, for an ncu metrics pass (dram bytes per launch -> profiles/traffic.json).

    python tools/profile_all.py            # prints the config order
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2311_07602_b200 import Context, workloads as W  # noqa: E402

CONFIGS = ["cfg1", "cfg2"] + [f"cfg3_b{b}_r{r}" for b in W.CFG3_B for r in W.CFG3_R] + [
    "cfg4", "cfg5"]


def main():
    ctx = Context(0)
    for name in CONFIGS:
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
            plan = ctx.ptr_plan("C", "N", "N", w.bs, w.rs, w.bs, pa, w.bs, pb, w.bs, pc, w.bs, 0.0)
            plan.execute()
            ctx.synchronize()
            print(f"{name} launches={plan.launches}", flush=True)
            del plan, arena
            continue
        count = w.batch
        if name == "cfg5":
            count = 16384  # one GPU's share at 8 GPUs (the whole batch does not fit)
        A, B, Cd = ctx.empty(w.sA * count), ctx.empty(w.sB * count), ctx.empty(w.sC * count)
        ctx.fill_uniform(A, w.a_rows, w.a_cols, w.lda, w.sA, count, w.seed, W.ROLE_A)
        ctx.fill_uniform(B, w.b_rows, w.b_cols, w.ldb, w.sB, count, w.seed, W.ROLE_B)
        ctx.dgemm_strided_batched(w.order, w.opA, w.opB, w.m, w.n, w.k, 0.0, A, w.lda, w.sA, B,
                                  w.ldb, w.sB, Cd, w.ldc, w.sC, count)
        ctx.synchronize()
        print(f"{name} launches=1 items={count}", flush=True)
        del A, B, Cd


if __name__ == "__main__":
    main()
