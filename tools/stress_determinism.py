#!/usr/bin/env python3
"""Repeat every producer/consumer pipeline form many times and require the
outputs to stay bitwise identical (catches ordering races that a single run
can miss): the panel kernel (producer warpgroup), a producer-warp tile
variant (n32), the warpgroup-producer s96, the release-counter q64 with its
TMA-store epilogue, the fused low-rank kernel (r = 8 producer, r = 32
release counter), and the BLR matvec (row problem with its deferred wait).

    python tools/stress_determinism.py [reps]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_07602_b200 import Context, DenseBlock  # noqa: E402
from paper_2311_07602_b200 import blr as B  # noqa: E402
from paper_2311_07602_b200 import lowrank as L  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    ctx = Context(0)
    rng = np.random.default_rng(1)
    bad = 0
    cases = [("p256", "C", "N", "T", 512, 512, 32, 400),
             ("n32", "C", "N", "N", 1024, 32, 1024, 300),
             ("s96", "C", "N", "N", 96, 96, 512, 2000),
             ("q64", "C", "N", "T", 512, 512, 8, 400)]
    for v, order, oa, ob, m, n, k, batch in cases:
        ra, ca = (k, m) if oa == "T" else (m, k)
        rb, cb = (n, k) if ob == "T" else (k, n)
        A = ctx.to_device(rng.uniform(-1, 1, ra * ca * batch))
        Bm = ctx.to_device(rng.uniform(-1, 1, rb * cb * batch))
        C = ctx.empty(m * n * batch)
        ctx.set_variant_override(v)
        first = None
        for _ in range(reps):
            ctx.dgemm_strided_batched(order, oa, ob, m, n, k, 0.0, A, ra, ra * ca, Bm, rb, rb * cb,
                                      C, m, m * n, batch)
            ctx.synchronize()
            got = C.download(m * n * batch)
            if first is None:
                first = got
                used = ctx.last_variant
            elif not np.array_equal(got, first):
                bad += 1
                print(f"FAIL {v}: run differs", flush=True)
                break
        ctx.set_variant_override(None)
        print(f"{v} (ran {used}): {reps} runs bitwise identical" if first is not None else v,
              flush=True)
    for r, blk in ((8, 1024), (32, 512)):
        lb = L.LowRankBatch.random(2000, blk, r, 7)
        ref = None
        for _ in range(max(1, reps // 5)):
            L.fused_multiply(lb, ctx=ctx)
            if ref is None:
                ref = lb.g_xy_batch.copy()
            elif not np.array_equal(lb.g_xy_batch, ref):
                bad += 1
                print(f"FAIL lowrank r={r}", flush=True)
                break
        print(f"lowrank r={r} block={blk}: repeated runs identical", flush=True)
    mat = B.BlrMatrix.random(64 * 32, 64, 8, 3)
    rhs = DenseBlock(64 * 32, 8, rng.uniform(-1, 1, 64 * 32 * 8))
    ref = None
    for _ in range(max(1, reps // 5)):
        y = B.blr_matvec(mat, rhs, ctx=ctx)
        if ref is None:
            ref = y.data.copy()
        elif not np.array_equal(y.data, ref):
            bad += 1
            print("FAIL blr matvec", flush=True)
            break
    print("blr matvec: repeated runs identical", flush=True)
    print(f"{bad} failures", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
