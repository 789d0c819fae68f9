#!/usr/bin/env python3
"""One launch of the auto-selected kernel per BASELINE config, in a fixed
order, for an ncu metrics pass (dram bytes per launch -> profiles/traffic.json).

    python tools/profile_all.py            # prints the config order
    python tools/profile_all.py --only blrd_n16384_b512_r16   # one row (full ncu capture)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2311_07602_b200 import Context, workloads as W  # noqa: E402

CONFIGS = ["cfg1", "cfg2"] + [f"cfg3_b{b}_r{r}" for b in W.CFG3_B for r in W.CFG3_R] + [
    "cfg4", "cfg5"]
# the widened rows (bench.py --config): low-rank product and BLR matvec
LOWRANK = ["lr_r8_b1024", "lr_r16_b1024", "lr_r32_b2048", "lr_r64_b2048", "lr_r96_b1024", "lr_r128_b1024"]
BLR = ["blr_n32768_b512_r8_k8", "blr_n16384_b256_r16_k16", "blr_n16384_b512_r32_k16"]
EXPAND = ["lrx_m512_r8", "lrx_m512_r32", "blrd_n16384_b512_r16"]


def expand_one(ctx, name):
    from paper_2311_07602_b200 import blr as BL

    w = W.get(name)
    if isinstance(w, W.BlrDense):
        mat = BL.BlrMatrix.random(w.n, w.block, w.rank, w.seed)
        out = ctx.empty(w.n * w.n)
        run = lambda: mat.reconstruct_dense_device(ctx, out)  # noqa: E731
    else:
        m, r, n = w.m, w.rank, w.batch
        bufs = [ctx.empty(n * m * r), ctx.empty(n * r * r), ctx.empty(n * r * m)]
        for b_ in bufs:
            b_.fill_bytes(0)
        out = ctx.empty(n * m * m)
        run = lambda: BL.lowrank_expand_device(ctx, n, m, m, r, *bufs, out)  # noqa: E731
    n0 = ctx.launch_count
    run()
    ctx.synchronize()
    print(f"{name}_warm launches={ctx.launch_count - n0}", flush=True)
    n0 = ctx.launch_count
    run()
    ctx.synchronize()
    print(f"{name} launches={ctx.launch_count - n0}", flush=True)


def lowrank_one(ctx, name):
    from paper_2311_07602_b200 import lowrank as L

    w = W.get_lowrank(name)
    n, r, blk = w.batch, w.rank, w.block
    bufs = [ctx.empty(n * r * blk), ctx.empty(n * blk * r), ctx.empty(n * r * r),
            ctx.empty(n * r * r), ctx.empty(n * r * r)]
    for i, (rows, cols) in enumerate(((blk, r), (r, blk), (r, r), (r, r))):
        ctx.fill_uniform(bufs[i], rows, cols, rows, rows * cols, n, w.seed, i, 0)
    n0 = ctx.launch_count
    L.lowrank_multiply_device(ctx, n, blk, r, *bufs)  # sizes the workspace (r > 32)
    ctx.synchronize()
    print(f"{name}_warm launches={ctx.launch_count - n0}", flush=True)
    n0 = ctx.launch_count
    L.lowrank_multiply_device(ctx, n, blk, r, *bufs)
    ctx.synchronize()
    print(f"{name} launches={ctx.launch_count - n0}", flush=True)


def blr_one(ctx, name, repeat=1):
    import bench_rows as R
    from paper_2311_07602_b200.lrbatch import _check, lib

    w = W.get_blr(name)
    m, rhs = R.blr_host(w)
    h = m.device_handle(ctx)
    d_rhs, d_y = ctx.to_device(rhs.data), ctx.empty(w.n * w.nrhs)
    run = lambda: _check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, w.nrhs, d_y.ptr, None),  # noqa
                         ctx._h)
    n0 = ctx.launch_count
    run()
    ctx.synchronize()
    print(f"{name}_warm launches={ctx.launch_count - n0}", flush=True)
    n0 = ctx.launch_count
    for _ in range(repeat):  # > 1: back-to-back launches (warm-cache traffic with --cache-control none)
        run()
    ctx.synchronize()
    print(f"{name} launches={ctx.launch_count - n0}", flush=True)
    m.invalidate()


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=None, help="config / row names (default: all)")
    ap.add_argument("--repeat", type=int, default=1, help="BLR matvec: launches after the warm-up")
    args = ap.parse_args()
    keep = (lambda n: True) if not args.only else (lambda n: n in args.only)
    ctx = Context(0)
    for name in filter(keep, CONFIGS):
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
            print(f"{name} launches={plan.launches} items={w.batch}", flush=True)
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
    for name in filter(keep, LOWRANK):
        lowrank_one(ctx, name)
    for name in filter(keep, BLR):
        blr_one(ctx, name, args.repeat)
    for name in filter(keep, EXPAND):
        expand_one(ctx, name)


if __name__ == "__main__":
    main()
