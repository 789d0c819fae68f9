#!/usr/bin/env python3
"""Small calls through every kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \\
        python tools/sanitize_cases.py

Strided GEMM (every variant, both loaders, ragged shapes, beta 1), a
pointer-array plan, the low-rank product (fused, three-GEMM and per-item
paths), BLR matvec and reconstruction, the low-rank expansion, the RNG fill,
LRBATCH1 device loads and a CUDA-graph replay. Exit 0 when every result
matches the FMA-chain oracle bitwise."""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2311_07602_b200 import Context, DenseBlock, variant_names  # noqa: E402
from paper_2311_07602_b200 import blr as B  # noqa: E402
from paper_2311_07602_b200 import lowrank as L  # noqa: E402

bad = 0


def check(name, ok):
    global bad
    print(("PASS " if ok else "FAIL ") + name, flush=True)
    bad += not ok


def main():
    ctx = Context(0)
    rng = np.random.default_rng(5)
    # strided GEMM: every variant, both loaders, ragged, beta 0 and 1
    m, n, k, batch = 70, 45, 37, 3
    A = rng.uniform(-1, 1, m * k * batch)
    Bm = rng.uniform(-1, 1, k * n * batch)
    C0 = rng.uniform(-1, 1, m * n * batch)
    dA, dB = ctx.to_device(A), ctx.to_device(Bm)
    for v in variant_names():
        ctx.set_variant_override(v)
        for loader in ("tma", "segment"):
            ctx.set_loader(loader)
            for beta in (0.0, 1.0):
                dC = ctx.to_device(C0)
                ctx.dgemm_strided_batched("C", "N", "N", m, n, k, beta, dA, m, m * k, dB, k, k * n,
                                          dC, m, m * n, batch)
                want = C0.copy()
                O.dgemm_strided("C", "N", "N", m, n, k, beta, A, m, m * k, Bm, k, k * n, want, m,
                                m * n, batch)
                check(f"gemm {v} {loader} beta={beta}", np.array_equal(dC.download(), want))
    ctx.set_variant_override(None)
    ctx.set_loader(None)
    # the row-panel kernel (short k, U V^T): k = 32 and a k-tail, beta 0 and 1
    for kp, beta in ((32, 0.0), (13, 1.0)):
        mp, np_, bp = 300, 70, 3
        Up = rng.uniform(-1, 1, mp * kp * bp)
        Vp = rng.uniform(-1, 1, np_ * kp * bp)
        Cp = rng.uniform(-1, 1, mp * np_ * bp)
        dC = ctx.to_device(Cp)
        ctx.set_variant_override("p256")
        ctx.dgemm_strided_batched("C", "N", "T", mp, np_, kp, beta, ctx.to_device(Up), mp, mp * kp,
                                  ctx.to_device(Vp), np_, np_ * kp, dC, mp, mp * np_, bp)
        ran = ctx.last_variant
        ctx.set_variant_override(None)
        want = Cp.copy()
        O.dgemm_strided("C", "N", "T", mp, np_, kp, beta, Up, mp, mp * kp, Vp, np_, np_ * kp, want,
                        mp, mp * np_, bp)
        check(f"panel k={kp} beta={beta}", ran == "p256" and np.array_equal(dC.download(), want))
    # pointer-array plan (variable sizes)
    ms, ns, ks = [64, 33, 130], [16, 40, 8], [64, 77, 130]
    As = [rng.uniform(-1, 1, a * c) for a, c in zip(ms, ks)]
    Bs = [rng.uniform(-1, 1, c * b) for c, b in zip(ks, ns)]
    dAs, dBs = [ctx.to_device(a) for a in As], [ctx.to_device(b) for b in Bs]
    dCs = [ctx.empty(a * b) for a, b in zip(ms, ns)]
    plan = ctx.ptr_plan("C", "N", "N", ms, ns, ks, dAs, ms, dBs, ks, dCs, ms, 0.0)
    plan.execute()
    ok = True
    for i in range(3):
        want = np.zeros(ms[i] * ns[i])
        O.dgemm_strided("C", "N", "N", ms[i], ns[i], ks[i], 0.0, As[i], ms[i], 0, Bs[i], ks[i], 0,
                        want, ms[i], 0, 1)
        ok = ok and np.array_equal(dCs[i].download(), want)
    check("pointer plan", ok)
    # the low-rank product: fused (r 8/16/32), three GEMMs (r 64), per-item (odd r)
    for r, blk in ((8, 64), (16, 96), (32, 64), (64, 128), (5, 17)):
        b = L.LowRankBatch.random(3, blk, r, r + blk)
        L.fused_multiply(b, ctx=ctx)
        fma = O.lowrank(3, blk, r, b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)
        check(f"lowrank r={r} block={blk}", np.array_equal(b.g_xy_batch, fma))
    # BLR matvec and reconstruction
    mat = B.BlrMatrix.random(96, 32, 6, 3)
    rhs = DenseBlock(96, 3, rng.uniform(-1, 1, 288))
    y = B.blr_matvec(mat, rhs, ctx=ctx)
    d, u, x, vt = mat.packed_arrays()
    check("blr matvec", np.array_equal(y.data, O.blr_matvec(96, 32, 6, d, u, x, vt, rhs.data, 3)))
    full = mat.reconstruct_dense(ctx=ctx)
    check("blr reconstruct", np.array_equal(full.data, O.blr_reconstruct(96, 32, 6, d, u, x, vt)))
    mat.invalidate()
    # BLR with b a multiple of 64 and even nrhs: the two-source row step and
    # the 4-D TMA-store reconstruction
    mat = B.BlrMatrix.random(192, 64, 8, 4)
    rhs = DenseBlock(192, 8, rng.uniform(-1, 1, 192 * 8))
    y = B.blr_matvec(mat, rhs, ctx=ctx)
    d, u, x, vt = mat.packed_arrays()
    check("blr matvec (row problem)",
          np.array_equal(y.data, O.blr_matvec(192, 64, 8, d, u, x, vt, rhs.data, 8)))
    full = mat.reconstruct_dense(ctx=ctx)
    check("blr reconstruct (tile problem)",
          np.array_equal(full.data, O.blr_reconstruct(192, 64, 8, d, u, x, vt)))
    mat.invalidate()
    # low-rank expansion
    u2, x2, v2 = (rng.uniform(-1, 1, s) for s in (2 * 40 * 6, 2 * 36, 2 * 6 * 30))
    got = B.lowrank_expand(u2, x2, v2, 2, 40, 30, 6, ctx=ctx)
    check("lowrank expand", np.array_equal(got, O.lowrank_expand(2, 40, 30, 6, u2, x2, v2)))
    # RNG fill
    buf = ctx.empty(50 * 7 * 2)
    ctx.fill_uniform(buf, 50, 7, 50, 350, 2, 9, 0)
    check("fill", np.array_equal(buf.download(), O.fill_uniform(50, 7, 50, 350, 2, 9, 0)))
    # LRBATCH1 into device memory
    lb = L.LowRankBatch.random(4, 32, 4, 8)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "b.lrb")
        L.save_batch(lb, path)
        _, bufs, _ = L.load_batch_device(ctx, path)
        check("batch file -> device", np.array_equal(bufs[0].download(), lb.a_vt_batch))
    # graph replay
    s = ctx.stream()
    dC = ctx.empty(m * n * batch)
    with ctx.capture(s) as cap:
        ctx.dgemm_strided_batched("C", "N", "N", m, n, k, 0.0, dA, m, m * k, dB, k, k * n, dC, m,
                                  m * n, batch, stream=s)
    cap.graph.launch(s)
    s.synchronize()
    want = np.zeros(m * n * batch)
    O.dgemm_strided("C", "N", "N", m, n, k, 0.0, A, m, m * k, Bm, k, k * n, want, m, m * n, batch)
    check("graph replay", np.array_equal(dC.download(), want))
    ctx.close()
    print(f"{bad} failures", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
