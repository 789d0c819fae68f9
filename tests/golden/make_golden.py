#!/usr/bin/env python3
"""Generate tests/golden/ from the REFERENCE ITSELF (oracle/_ref/liblrb_ref.so,
compiled from /root/reference/proj/include/lrbatch/dense.hpp by `make ref`).

Run here (where /root/reference exists):  python tests/golden/make_golden.py

Outputs
  gemm_golden.npz    inputs + reference outputs for small seeded cases (row-major
                     gemm_naive_raw calls, and column-major batches through the
                     operand swap of SURVEY.md §0), plus sha256 digests of the
                     outputs of BASELINE-shaped batches (too large to store)
  shape_errors.json  dense_gemm_naive's ShapeError texts (dense.hpp:58-69)

Inputs come from the counter RNG of include/lrb_rng.h (oracle.fill_uniform), so
the tests regenerate them bit-for-bit; the stored copies guard the RNG too.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

# (name, order, opA, opB, m, n, k, batch, accumulate, seed)
SMALL = [
    ("rm_1x1x1", "R", "N", "N", 1, 1, 1, 1, 0, 10),
    ("rm_3x7x5", "R", "N", "N", 3, 7, 5, 1, 0, 11),
    ("rm_17x5x13_acc", "R", "N", "N", 17, 5, 13, 1, 1, 12),
    ("rm_64x64x64", "R", "N", "N", 64, 64, 64, 1, 0, 13),
    ("rm_33x16x257", "R", "N", "N", 33, 16, 257, 2, 0, 14),
    ("cm_nn_37x11x29", "C", "N", "N", 37, 11, 29, 3, 0, 20),
    ("cm_nt_41x19x23", "C", "N", "T", 41, 19, 23, 3, 0, 21),
    ("cm_tn_23x9x31_acc", "C", "T", "N", 23, 9, 31, 2, 1, 22),
    ("cm_tt_12x40x7", "C", "T", "T", 12, 40, 7, 2, 0, 23),
    ("cm_nn_256x16x256", "C", "N", "N", 256, 16, 256, 2, 0, 0),  # cfg1 shape, seed 0
    ("cm_nt_64x64x32", "C", "N", "T", 64, 64, 32, 2, 0, 1),      # cfg2 shape class
]
# BASELINE-shaped batches: stored as digests of the reference output
DIGEST = [
    ("cfg1_full", "C", "N", "N", 256, 16, 256, 256, 0, 0),
    ("cfg2_items0_3", "C", "N", "T", 512, 512, 32, 4, 0, 1),
    ("cfg3_b512_r32_items0_1", "C", "N", "N", 512, 32, 512, 2, 0, 2),
    ("cfg5_items0_1", "C", "N", "N", 512, 32, 512, 2, 0, 4),
]


def stored(order, op, r, c):
    s = (c, r) if op == "T" else (r, c)
    return s if order == "C" else (s[1], s[0])  # column-major view (rows, cols)


def make_inputs(order, opA, opB, m, n, k, batch, acc, seed):
    ar, ac = stored(order, opA, m, k)
    br, bc = stored(order, opB, k, n)
    cr, cc = stored(order, "N", m, n)
    A = O.fill_uniform(ar, ac, ar, ar * ac, batch, seed, 0)
    B = O.fill_uniform(br, bc, br, br * bc, batch, seed, 1)
    C0 = O.fill_uniform(cr, cc, cr, cr * cc, batch, seed, 2) if acc else np.zeros(cr * cc * batch)
    return A, B, C0, (ar, ac), (br, bc), (cr, cc)


def reference(order, opA, opB, m, n, k, batch, acc, A, B, C0, sa, sb, sc):
    out = C0.copy()
    if order == "R":
        assert opA == "N" and opB == "N"
        for it in range(batch):
            a = np.ascontiguousarray(A[it * m * k:(it + 1) * m * k])
            b = np.ascontiguousarray(B[it * k * n:(it + 1) * k * n])
            c = np.ascontiguousarray(out[it * m * n:(it + 1) * m * n])
            O.ref_gemm_naive_raw(a, b, c, m, k, n, acc)
            out[it * m * n:(it + 1) * m * n] = c
    else:
        O.ref_dgemm_colmajor(opA, opB, m, n, k, acc, A, sa[0], sa[0] * sa[1], B, sb[0],
                             sb[0] * sb[1], out, sc[0], sc[0] * sc[1], batch, threads=8)
    return out


def main():
    if not O.ref_available():
        sys.exit("oracle/_ref/liblrb_ref.so missing: run `make ref` where /root/reference exists")
    arrays = {}
    meta = {"small": [], "digest": []}
    for case in SMALL:
        name = case[0]
        A, B, C0, sa, sb, sc = make_inputs(*case[1:])
        out = reference(*case[1:9], A, B, C0, sa, sb, sc)
        arrays[f"{name}__A"] = A
        arrays[f"{name}__B"] = B
        arrays[f"{name}__C0"] = C0
        arrays[f"{name}__C"] = out
        meta["small"].append(list(case))
    for case in DIGEST:
        name = case[0]
        A, B, C0, sa, sb, sc = make_inputs(*case[1:])
        out = reference(*case[1:9], A, B, C0, sa, sb, sc)
        meta["digest"].append(list(case) + [hashlib.sha256(out.tobytes()).hexdigest(),
                                            float(out[0]), float(out[-1])])
    # flops counter of the reference (2 per multiply-add, dense.hpp:148)
    a = O.fill_uniform(7, 9, 7, 63, 1, 5, 0)
    b = O.fill_uniform(9, 5, 9, 45, 1, 5, 1)
    c = np.zeros(35)
    fl = np.zeros(1, dtype=np.uint64)
    O.ref_gemm_naive_raw(a, b, c, 7, 9, 5, False, fl)
    arrays["flops__A"], arrays["flops__B"], arrays["flops__C"] = a, b, c
    meta["flops"] = {"m": 7, "k": 9, "n": 5, "count": int(fl[0])}
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "gemm_golden.npz"), **arrays)

    errors = []
    for (ar, ac, br, bc, orow, ocol) in [(2, 3, 4, 2, 2, 2), (2, 3, 3, 2, 3, 3), (1, 5, 5, 1, 2, 1),
                                         (4, 4, 4, 4, 4, 5), (3, 0, 1, 2, 3, 2)]:
        msg = O.ref_dense_gemm_naive_error(ar, ac, br, bc, orow, ocol)
        errors.append({"a": [ar, ac], "b": [br, bc], "out": [orow, ocol], "error": msg})
    with open(os.path.join(HERE, "shape_errors.json"), "w") as f:
        json.dump(errors, f, indent=1)
    print(f"wrote {len(SMALL)} small cases, {len(DIGEST)} digests, {len(errors)} error texts")


if __name__ == "__main__":
    main()
