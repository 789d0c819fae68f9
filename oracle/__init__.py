"""CPU oracle for the batched FP64 GEMM hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. It is the checker, never the
product: paper_2311_07602_b200 does not import it and has no CPU fallback.

Two libraries:
  * ``liblrb_oracle.so`` — the C restatement (oracle/lrb_oracle.c) of the
    reference's gemm_naive_raw (proj/include/lrbatch/dense.hpp:43-56);
  * ``_ref/liblrb_ref.so`` — the reference itself compiled from
    /root/reference by the Makefile's ``ref`` target (travels prebuilt to the
    GPU box; the reference tree does not).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblrb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblrb_ref.so")

FMA_CHAIN = 0      # one fma() per k step (the device kernels' rounding)
REF_COMPILED = 1   # the reference binary's rounding

i64, dbl, vp = C.c_int64, C.c_double, C.c_void_p
P = C.POINTER

_oracle = None
_ref = None


def oracle_lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make oracle`")
        L = C.CDLL(ORACLE_SO)
        L.oracle_gemm_naive_raw.argtypes = [vp, vp, vp, C.c_size_t, C.c_size_t, C.c_size_t,
                                            C.c_int, P(C.c_uint64)]
        L.oracle_gemm_naive_raw.restype = None
        L.oracle_dgemm_strided.argtypes = [C.c_int, C.c_char, C.c_char, C.c_char, i64, i64, i64,
                                           dbl, vp, i64, i64, vp, i64, i64, vp, i64, i64, i64,
                                           C.c_int]
        L.oracle_dgemm_strided.restype = C.c_int
        L.oracle_dgemm_ptr.argtypes = [C.c_int, C.c_char, C.c_char, C.c_char, i64, P(i64), P(i64),
                                       P(i64), P(vp), P(i64), P(vp), P(i64), P(vp), P(i64), dbl,
                                       C.c_int]
        L.oracle_dgemm_ptr.restype = C.c_int
        L.oracle_fill_uniform.argtypes = [vp, i64, i64, i64, i64, i64, C.c_uint64, C.c_uint32, i64]
        L.oracle_fill_uniform.restype = None
        L.oracle_check_bound.argtypes = [C.c_char, C.c_char, C.c_char, i64, i64, i64, dbl, vp, i64,
                                         vp, i64, vp, vp, vp, i64, P(dbl)]
        L.oracle_check_bound.restype = i64
        L.oracle_lowrank_batch.argtypes = [C.c_int, i64, i64, i64, vp, vp, vp, vp, vp, C.c_int]
        L.oracle_lowrank_batch.restype = C.c_int
        L.oracle_blr_matvec.argtypes = [C.c_int, i64, i64, i64, vp, vp, vp, vp, vp, i64, vp]
        L.oracle_lowrank_expand.argtypes = [C.c_int, i64, i64, i64, i64, vp, i64, vp, i64, vp,
                                            i64, vp, i64, i64]
        L.oracle_lowrank_expand.restype = C.c_int
        L.oracle_blr_reconstruct.argtypes = [C.c_int, i64, i64, i64, vp, vp, vp, vp, vp]
        L.oracle_blr_reconstruct.restype = C.c_int
        L.oracle_blr_matvec.restype = C.c_int
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise ImportError(f"{REF_SO} missing: run `make ref` where /root/reference exists")
        L = C.CDLL(REF_SO)
        L.ref_gemm_naive_raw.argtypes = [vp, vp, vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int,
                                         P(C.c_uint64)]
        L.ref_gemm_naive_raw.restype = None
        L.ref_gemm_rowmajor_batched.argtypes = [vp, vp, vp, C.c_size_t, C.c_size_t, C.c_size_t,
                                                C.c_int, i64, C.c_int]
        L.ref_gemm_rowmajor_batched.restype = None
        L.ref_dgemm_colmajor_strided.argtypes = [C.c_char, C.c_char, i64, i64, i64, C.c_int, vp,
                                                 i64, i64, vp, i64, i64, vp, i64, i64, i64,
                                                 C.c_int]
        L.ref_dgemm_colmajor_strided.restype = C.c_int
        L.ref_dgemm_colmajor_ptr.argtypes = [C.c_char, C.c_char, i64, P(i64), P(i64), P(i64),
                                             P(vp), P(i64), P(vp), P(i64), P(vp), P(i64), C.c_int,
                                             C.c_int]
        L.ref_dgemm_colmajor_ptr.restype = C.c_int
        L.ref_dense_gemm_naive_error.argtypes = [C.c_size_t] * 6 + [C.c_char_p, C.c_size_t]
        L.ref_dense_gemm_naive_error.restype = C.c_int
        L.ref_lowrank_multiply.argtypes = [C.c_int, i64, i64, i64, vp, vp, vp, vp, vp, C.c_int,
                                           C.c_char_p, P(i64)]
        L.ref_lowrank_multiply.restype = C.c_int
        L.ref_compare_to_reference.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, P(i64), P(i64)]
        L.ref_compare_to_reference.restype = dbl
        L.ref_blr_matvec.argtypes = [C.c_int, i64, i64, i64, vp, vp, vp, vp, vp, i64, vp, C.c_int,
                                     C.c_char_p, P(i64)]
        L.ref_blr_matvec.restype = C.c_int
        L.ref_blr_reconstruct.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp]
        L.ref_blr_reconstruct.restype = C.c_int
        L.ref_lowrank_expand.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, C.c_int]
        L.ref_lowrank_expand.restype = C.c_int
        L.ref_bench_csv_header.argtypes = [C.c_char_p, C.c_size_t]
        L.ref_bench_csv_header.restype = C.c_int
        L.ref_bench_csv_row.argtypes = [vp, C.c_char_p, C.c_size_t]
        L.ref_bench_csv_row.restype = C.c_int
        L.ref_bench_rates.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, dbl, vp]
        L.ref_bench_rates.restype = C.c_int
        L.ref_median_of.argtypes = [vp, i64]
        L.ref_median_of.restype = dbl
        L.ref_last_seconds.argtypes = []
        L.ref_last_seconds.restype = dbl
        L.ref_packing_plan.argtypes = [C.c_char_p, i64, i64, P(i64)]
        L.ref_packing_plan.restype = C.c_int
        _ref = L
    return _ref


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


# ------------------------------------------------------------------ oracle
def gemm_naive_raw(a, b, c, m, k, n, accumulate, flops: Optional[np.ndarray] = None):
    fl = C.c_uint64(int(flops[0]) if flops is not None else 0)
    oracle_lib().oracle_gemm_naive_raw(_p(a), _p(b), _p(c), m, k, n, int(bool(accumulate)),
                                       C.byref(fl) if flops is not None else None)
    if flops is not None:
        flops[0] = fl.value


def dgemm_strided(order, opA, opB, m, n, k, beta, A, lda, sA, B, ldb, sB, Cm, ldc, sC, batch,
                  threads=1, mode=FMA_CHAIN):
    rc = oracle_lib().oracle_dgemm_strided(mode, order.encode(), opA.encode(), opB.encode(), m, n,
                                           k, float(beta), _p(A), lda, sA, _p(B), ldb, sB, _p(Cm),
                                           ldc, sC, batch, threads)
    if rc != 0:
        raise ValueError("oracle_dgemm_strided: bad arguments")


def _arr64(xs):
    a = np.ascontiguousarray(np.asarray(xs, dtype=np.int64))
    return a, a.ctypes.data_as(P(i64))


def dgemm_ptr(order, opA, opB, m, n, k, A, lda, B, ldb, Cs, ldc, beta, threads=1, mode=FMA_CHAIN):
    batch = len(m)
    keep = [_arr64(x) for x in (m, n, k, lda, ldb, ldc)]
    pa = (vp * batch)(*[_p(x) for x in A])
    pb = (vp * batch)(*[_p(x) for x in B])
    pc = (vp * batch)(*[_p(x) for x in Cs])
    rc = oracle_lib().oracle_dgemm_ptr(mode, order.encode(), opA.encode(), opB.encode(), batch,
                                       keep[0][1], keep[1][1], keep[2][1], pa, keep[3][1], pb,
                                       keep[4][1], pc, keep[5][1], float(beta), threads)
    if rc != 0:
        raise ValueError("oracle_dgemm_ptr: bad arguments")


def fill_uniform(rows, cols, ld, stride, batch, seed, role, item_offset=0) -> np.ndarray:
    n = stride * (batch - 1) + ld * (cols - 1) + rows if batch and rows and cols else 0
    out = np.zeros(max(n, 0), dtype=np.float64)
    if n:
        oracle_lib().oracle_fill_uniform(_p(out), rows, cols, ld, stride, batch, seed, role,
                                         item_offset)
    return out


def check_bound(order, opA, opB, m, n, k, beta, A, lda, B, ldb, C0, Cm, Cref, ldc):
    """(violations, max err/bound) of BASELINE's componentwise bound for one item."""
    ratio = C.c_double(0.0)
    bad = oracle_lib().oracle_check_bound(order.encode(), opA.encode(), opB.encode(), m, n, k,
                                          float(beta), _p(A), lda, _p(B), ldb,
                                          _p(C0) if C0 is not None else None, _p(Cm), _p(Cref),
                                          ldc, C.byref(ratio))
    return int(bad), float(ratio.value)


# --------------------------------------------------------------- reference
def ref_gemm_naive_raw(a, b, c, m, k, n, accumulate, flops: Optional[np.ndarray] = None):
    fl = C.c_uint64(int(flops[0]) if flops is not None else 0)
    ref_lib().ref_gemm_naive_raw(_p(a), _p(b), _p(c), m, k, n, int(bool(accumulate)),
                                 C.byref(fl) if flops is not None else None)
    if flops is not None:
        flops[0] = fl.value


def ref_dgemm_colmajor(opA, opB, m, n, k, accumulate, A, lda, sA, B, ldb, sB, Cm, ldc, sC, batch,
                       threads=1):
    rc = ref_lib().ref_dgemm_colmajor_strided(opA.encode(), opB.encode(), m, n, k,
                                              int(bool(accumulate)), _p(A), lda, sA, _p(B), ldb,
                                              sB, _p(Cm), ldc, sC, batch, threads)
    if rc != 0:
        raise ValueError("ref_dgemm_colmajor_strided: bad arguments")


def ref_dgemm_colmajor_ptr(opA, opB, m, n, k, A, lda, B, ldb, Cs, ldc, accumulate, threads=1):
    batch = len(m)
    keep = [_arr64(x) for x in (m, n, k, lda, ldb, ldc)]
    pa = (vp * batch)(*[_p(x) for x in A])
    pb = (vp * batch)(*[_p(x) for x in B])
    pc = (vp * batch)(*[_p(x) for x in Cs])
    ref_lib().ref_dgemm_colmajor_ptr(opA.encode(), opB.encode(), batch, keep[0][1], keep[1][1],
                                     keep[2][1], pa, keep[3][1], pb, keep[4][1], pc, keep[5][1],
                                     int(bool(accumulate)), threads)


def ref_rowmajor_batched(a, b, c, m, k, n, accumulate, batch, threads=1):
    ref_lib().ref_gemm_rowmajor_batched(_p(a), _p(b), _p(c), m, k, n, int(bool(accumulate)),
                                        batch, threads)


def ref_dense_gemm_naive_error(ar, ac, br, bc, orow, ocol) -> Optional[str]:
    buf = C.create_string_buffer(256)
    if ref_lib().ref_dense_gemm_naive_error(ar, ac, br, bc, orow, ocol, buf, 256):
        return buf.value.decode()
    return None


# ------------------------------------------------------- low-rank product
def lowrank(batch, block, rank, a_vt, b_u, a_x, b_x, threads=1, mode=FMA_CHAIN):
    """G = A_X (A_Vt B_U) B_X per item (low_rank.hpp:73-87), rounded per `mode`"""
    g = np.zeros(batch * rank * rank)
    rc = oracle_lib().oracle_lowrank_batch(mode, batch, block, rank, _p(a_vt), _p(b_u), _p(a_x),
                                           _p(b_x), _p(g), threads)
    if rc != 0:
        raise ValueError("oracle_lowrank_batch: bad arguments")
    return g


# ------------------------------------------------- the reference's packing plans
# the plan the GPU box's Xeon host runs fastest (tools/probe_cpu_ref.py: 2.4x
# the epyc-7502 plan at r >= 32, equal at r = 8)
DEFAULT_MACHINE = "skylake-x-6148"
PLAN_FIELDS = ("b_small", "b_skinny", "m_pack", "n_pack", "x_pack", "y_pack", "tile", "llc_bytes",
               "alignment_bytes", "dual_accumulator")
_PLANS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                      "golden", "packing_plans.json")
_plan_cache = None


def ref_last_seconds() -> float:
    """wall time of the last ref_lowrank / ref_blr_matvec driver call alone
    (excludes copying the inputs into the reference's containers)"""
    return float(ref_lib().ref_last_seconds())


def ref_packing_plan_live(machine, rank, block=0):
    """make_packing_plan (plan.hpp:66-100) from the reference's machine files
    (only where /root/reference exists); None if the reference rejects it"""
    f = (C.c_int64 * 10)()
    rc = ref_lib().ref_packing_plan(machine.encode(), rank, block, f)
    return None if rc != 0 else [int(v) for v in f]


def packing_plan(machine=None, rank=8, block=0):
    """The reference's PackingPlan for (machine, rank) as 10 fields: live from
    its machine files when present, else the committed fixture
    tests/golden/packing_plans.json (made by tests/golden/make_plans.py from
    the same call). The plan depends on rank only (plan.hpp:68)."""
    global _plan_cache
    machine = machine or DEFAULT_MACHINE
    if ref_machines_available():
        return ref_packing_plan_live(machine, rank, block)
    if _plan_cache is None:
        with open(_PLANS) as fh:
            _plan_cache = json.load(fh)
    return _plan_cache["plans"][machine].get(str(rank))


def _plan_arg(machine, rank):
    fields = packing_plan(machine, rank)
    if fields is None:
        raise ValueError(f"no packing plan for machine {machine or DEFAULT_MACHINE} rank {rank}")
    return (C.c_int64 * 10)(*fields)


def ref_lowrank(which, batch, block, rank, a_vt, b_u, a_x, b_x, workers=1, machine=None):
    """the reference's own drivers: 0 naive_multiply_batch, 1 fused_multiply,
    2 packed_multiply (the reference's plan for `machine`, see packing_plan)"""
    g = np.zeros(batch * rank * rank)
    plan = _plan_arg(machine, rank) if which == 2 else None
    rc = ref_lib().ref_lowrank_multiply(which, batch, block, rank, _p(a_vt), _p(b_u), _p(a_x),
                                        _p(b_x), _p(g), workers, None, plan)
    if rc != 0:
        raise ValueError("ref_lowrank_multiply failed")
    return g


def ref_compare_to_reference(batch, block, rank, a_vt, b_u, a_x, b_x, g):
    """the reference's compare_to_reference metric (verify.hpp:38-64):
    (max relative error, worst item, worst entry)"""
    wi, we = C.c_int64(0), C.c_int64(0)
    err = ref_lib().ref_compare_to_reference(batch, block, rank, _p(a_vt), _p(b_u), _p(a_x),
                                             _p(b_x), _p(g), C.byref(wi), C.byref(we))
    return float(err), int(wi.value), int(we.value)


def lowrank_bound_check(batch, block, rank, a_vt, b_u, a_x, b_x, g, g_ref):
    """Componentwise bound for the chained product (three naive products):
    |G - G_ref| <= 4 (b + 2r) 2^-52 (|A_X| |A_Vt| |B_U| |B_X|), evaluated with
    the same chain on absolute values. Returns (violations, max ratio)."""
    mags = lowrank(batch, block, rank, np.abs(a_vt), np.abs(b_u), np.abs(a_x), np.abs(b_x),
                   threads=4)
    bound = 4.0 * (block + 2 * rank) * 2.0 ** -52 * mags
    err = np.abs(g - g_ref)
    exact = bound == 0
    bad = int(np.sum(err[~exact] > bound[~exact]) + np.sum(err[exact] != 0))
    ratio = float(np.max(err[~exact] / bound[~exact])) if np.any(~exact) else 0.0
    return bad, ratio


# ------------------------------------------------------------ BLR matvec
def blr_matvec(n, block, rank, diag, u, x, vt, rhs, nrhs, mode=FMA_CHAIN):
    """blr_matvec_naive (blr.hpp:179-202) rounded per `mode`"""
    y = np.zeros(n * nrhs)
    rc = oracle_lib().oracle_blr_matvec(mode, n, block, rank, _p(diag), _p(u), _p(x), _p(vt),
                                        _p(rhs), nrhs, _p(y))
    if rc != 0:
        raise ValueError("oracle_blr_matvec: bad arguments")
    return y


def ref_blr_matvec(which, n, block, rank, diag, u, x, vt, rhs, nrhs, workers=2, machine=None):
    """the reference itself: 0 blr_matvec (packed; plan at rank max(rank, nrhs)
    per blr.hpp), 1 blr_matvec_naive, 2 dense reconstruction"""
    y = np.zeros(n * nrhs)
    plan = _plan_arg(machine, max(rank, nrhs)) if which == 0 else None
    rc = ref_lib().ref_blr_matvec(which, n, block, rank, _p(diag), _p(u), _p(x), _p(vt), _p(rhs),
                                  nrhs, _p(y), workers, None, plan)
    if rc != 0:
        raise ValueError("ref_blr_matvec failed")
    return y


def lowrank_expand(batch, m, n, r, u, x, vt, mode=FMA_CHAIN, su=None, sx=None, svt=None,
                   ldo=None, so=None, out=None):
    """out_i = (U_i X_i) Vt_i (blr.hpp:75-78 per tile) rounded per `mode`"""
    su = m * r if su is None else su
    sx = r * r if sx is None else sx
    svt = r * n if svt is None else svt
    ldo = n if ldo is None else ldo
    so = m * ldo if so is None else so
    if out is None:
        out = np.zeros(max(1, (batch - 1) * so + max(0, (m - 1) * ldo + n)))
    rc = oracle_lib().oracle_lowrank_expand(mode, batch, m, n, r, _p(u), su, _p(x), sx, _p(vt),
                                            svt, _p(out), ldo, so)
    if rc != 0:
        raise ValueError("oracle_lowrank_expand: bad arguments")
    return out


def blr_reconstruct(n, block, rank, diag, u, x, vt, mode=FMA_CHAIN):
    """BlrMatrix::reconstruct_dense (blr.hpp:62-86) rounded per `mode`"""
    out = np.zeros(n * n)
    rc = oracle_lib().oracle_blr_reconstruct(mode, n, block, rank, _p(diag), _p(u), _p(x),
                                             _p(vt), _p(out))
    if rc != 0:
        raise ValueError("oracle_blr_reconstruct: bad arguments")
    return out


def ref_blr_reconstruct(n, block, rank, diag, u, x, vt):
    """the reference's own reconstruct_dense"""
    out = np.zeros(n * n)
    if ref_lib().ref_blr_reconstruct(n, block, rank, _p(diag), _p(u), _p(x), _p(vt), _p(out)):
        raise ValueError("ref_blr_reconstruct failed")
    return out


def ref_lowrank_expand(batch, m, n, r, u, x, vt, workers=1):
    """the reference's (U X) Vt per item through its gemm_naive_raw"""
    out = np.zeros(batch * m * n)
    if ref_lib().ref_lowrank_expand(batch, m, n, r, _p(u), _p(x), _p(vt), _p(out), workers):
        raise ValueError("ref_lowrank_expand failed")
    return out


def ref_bench_csv_header() -> str:
    """lrbatch::bench_csv_header (bench.hpp:125-129)"""
    buf = C.create_string_buffer(1024)
    if ref_lib().ref_bench_csv_header(buf, 1024):
        raise ValueError("ref_bench_csv_header failed")
    return buf.value.decode()


def ref_bench_csv_row(values) -> str:
    """lrbatch::bench_csv_row (bench.hpp:131-141) of 17 column values"""
    v = np.asarray(values, dtype=np.float64)
    buf = C.create_string_buffer(1024)
    if ref_lib().ref_bench_csv_row(_p(v), buf, 1024):
        raise ValueError("ref_bench_csv_row failed")
    return buf.value.decode()


def ref_bench_rates(batch, rank, block, seconds):
    """(gflops, bandwidth_overlapped_gib_s, bandwidth_nonoverlapped_gib_s), or None on ShapeError"""
    out = np.zeros(3)
    if ref_lib().ref_bench_rates(batch, rank, block, seconds, _p(out)):
        return None
    return tuple(float(x) for x in out)


def ref_median_of(values) -> float:
    v = np.asarray(values, dtype=np.float64)
    return float(ref_lib().ref_median_of(_p(v), v.size))


def ref_machines_available() -> bool:
    """the reference's packed drivers resolve CPU machine files from its own
    tree (LRBATCH_MACHINE_DIR); present only where /root/reference exists"""
    return os.path.isdir("/root/reference/proj/machines")
