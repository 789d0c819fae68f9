"""CPU: the C-ABI library (liblrb.so) and its host-side logic, no GPU needed.

* the in-tree library loads and exports exactly what include/lrb.h declares;
* argument validation (reference ShapeError semantics, dense.hpp:58-69) runs
  before any device work, so it is testable with a NULL context;
* the selector and the shard planner are host-only.
"""
import ctypes as C
import json
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2311_07602_b200 as P
from paper_2311_07602_b200 import _lib
from paper_2311_07602_b200._lib import lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "lrb.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lrb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    declared = set(declared_symbols())
    assert declared, "no declarations parsed"
    missing = declared - exported
    assert not missing, f"declared but not exported: {missing}"
    extra = {s for s in exported if not s.startswith("lrb_")}
    assert not extra, f"non-ABI symbols leak from liblrb.so: {sorted(extra)[:5]}"


def test_python_binding_covers_the_header():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_variants():
    assert P.version().startswith("lrb-b200")
    names = P.variant_names()
    assert {"n8", "n16", "n32", "n64", "sq", "m8", "m16", "m32", "m64"} <= set(names)
    for i, nm in enumerate(names):
        assert P.variant_from_name(nm) == i
    assert P.variant_from_name("nope") == -1


def test_no_device_here_fails_loudly():
    if P.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(P.NoDeviceError):
        P.Context(0)


# ----------------------------------------------------------------- selector
@pytest.mark.parametrize("m,n,k,want", [
    (256, 16, 256, "n16"), (512, 512, 32, "p256"), (512, 512, 48, "q64p"), (512, 512, 16, "q64"), (512, 32, 512, "n32"), (1024, 8, 1024, "n8"),
    (2048, 64, 2048, "t64"), (128, 64, 128, "n64"), (512, 24, 512, "n24"), (512, 40, 512, "n40"), (512, 48, 512, "n48"),
    (512, 56, 512, "n56"), (16, 512, 512, "m16k64"), (16, 512, 32, "m16"), (8, 300, 7, "m8"),
    (8, 300, 300, "m8k64"), (64, 200, 64, "m64"),
])
def test_selector_by_shape(m, n, k, want):
    batch = 100000
    s = P.select("C", "N", "N", m, n, k, batch)
    assert s["name"] == want
    assert s["tiles"] == batch * -(-m // s["tile_m"]) * -(-n // s["tile_n"])


def test_selector_small_skinny_batches_use_short_tiles():
    # cfg1: 256 items of 256 x 16 -> fewer than two waves of 128-row tiles
    assert P.select("C", "N", "N", 256, 16, 256, 256)["name"] == "n16t"
    assert P.select("C", "N", "N", 256, 16, 256, 100000)["name"] == "n16"
    # short-wide C with a short k and a small batch: 32-column tiles
    assert P.select("R", "N", "N", 512, 8, 32, 64)["name"] == "m8t"
    assert P.select("R", "N", "N", 256, 16, 48, 64)["name"] == "m16t"
    assert P.select("R", "N", "N", 256, 16, 48, 100000)["name"] == "m16"


def test_selector_row_major_long_k_uses_k64_tiles():
    # the row-major drop-in's big block is contiguous along k: 64-deep chunks
    assert P.select("R", "N", "N", 512, 8, 504, 64)["name"] == "m8k64"
    assert P.select("R", "N", "N", 256, 16, 1008, 64)["name"] == "m16k64"
    assert P.select("R", "N", "N", 1024, 16, 1024, 10000)["name"] == "m16k64"
    assert P.select("R", "N", "N", 512, 32, 512, 10000)["name"] == "m32"


def test_selector_long_k_general_shapes_use_t64():
    # 128 x 64 tiles with 64 x 32 warp tiles once k >= 128 (the low-rank
    # product's r = 128 GEMMs); short-k U V^T (cfg2) takes the row-panel
    # kernel, and q64p (q64 with a producer warp) where the panel does not
    # serve (k > 32, op(A) = T)
    assert P.select("R", "N", "N", 128, 128, 1024, 20000)["name"] == "t64"
    assert P.select("R", "N", "N", 128, 128, 128, 20000)["name"] == "t64"
    assert P.select("C", "N", "T", 512, 512, 32, 4096)["name"] == "p256"
    assert P.select("C", "N", "T", 512, 512, 33, 4096)["name"] == "q64p"
    assert P.select("C", "T", "T", 512, 512, 32, 4096)["name"] == "q64p"
    # too few 256-row units for one wave, or too short: the tile kernel
    assert P.select("C", "N", "T", 512, 512, 32, 50)["name"] == "q64p"
    # write-bound short k: the tile kernel's TMA-store epilogue
    assert P.select("C", "N", "T", 512, 512, 16, 4096)["name"] == "q64"
    assert P.select("C", "N", "T", 512, 512, 17, 4096)["name"] == "p256"
    assert P.select("C", "N", "T", 128, 512, 32, 4096)["name"] != "p256"
    assert P.select("R", "N", "N", 64, 64, 1024, 20000)["name"] == "q64q"
    assert P.select("R", "N", "N", 64, 64, 128, 20000)["name"] == "q64p"


def test_selector_rank96_uses_s96():
    # 96 x 96 outputs: s96 fits exactly where q64 / t64 pad to 128 x 128
    assert P.select("R", "N", "N", 96, 96, 1024, 20000)["name"] == "s96"
    assert P.select("R", "N", "N", 96, 96, 96, 20000)["name"] == "s96"
    assert P.select("C", "N", "N", 80, 80, 64, 1000)["name"] == "s96"
    assert P.select("C", "N", "T", 512, 512, 48, 4096)["name"] == "q64p"


def test_selector_row_major_swaps_roles():
    # row-major C (m x n) is column-major C^T (n x m): the reference's BLR
    # diagonal step D(b x b) * rhs(b x r) lands on the short-wide m-variants
    s = P.select("R", "N", "N", 1024, 16, 1024, 10000)
    assert s["name"] == "m16k64"
    assert P.select("R", "N", "N", 1024, 16, 32, 4)["name"] == "m16t"  # short k, < two waves


def test_selector_intensity_and_bound():
    s1 = P.select("C", "N", "N", 256, 16, 256, 256)
    assert abs(s1["intensity"] - 3.5556) < 1e-3 and not s1["fp64_bound"]
    s2 = P.select("C", "N", "T", 512, 512, 32, 4096)
    assert abs(s2["intensity"] - 7.1111) < 1e-3 and s2["fp64_bound"]


def test_selector_rejects_bad_input():
    with pytest.raises(P.ArgError):
        P.select("X", "N", "N", 1, 1, 1, 1)
    with pytest.raises(P.ShapeError):
        P.select("C", "N", "N", -1, 1, 1, 1)


# ------------------------------------------------------------ shard planner
def test_shard_plan_reference_split():
    # per = ceil(batch / parts), contiguous (reference bench.hpp:69-75)
    assert P.shard_plan(10, 3) == [0, 4, 8, 10]
    assert P.shard_plan(131072, 8) == [i * 16384 for i in range(9)]
    assert P.shard_plan(3, 8) == [0, 1, 2, 3, 3, 3, 3, 3, 3]
    assert P.shard_plan(0, 2) == [0, 0, 0]


def test_shard_plan_weighted_balances_cost():
    from paper_2311_07602_b200 import workloads as W

    w = W.get("cfg4")
    cost = [w.item_flops(i) for i in range(w.batch)]
    for parts in (2, 4, 8):
        b = P.shard_plan(w.batch, parts, cost)
        assert b[0] == 0 and b[-1] == w.batch and b == sorted(b)
        per = [sum(cost[b[g]:b[g + 1]]) for g in range(parts)]
        assert max(per) / (sum(per) / parts) < 1.01


def test_shard_plan_rejects_bad_cost():
    with pytest.raises(P.ArgError):
        P.shard_plan(3, 2, [1.0, -1.0, 1.0])
    with pytest.raises(P.ArgError):
        P.shard_plan(3, 0)


# --------------------------------------------------------------- validation
def _strided(order="C", opA="N", opB="N", m=4, n=3, k=2, beta=0.0, lda=4, sA=8, ldb=2, sB=6,
             ldc=4, sC=12, batch=2, ptrs=(16, 16, 16)):
    st = lib.lrb_dgemm_strided_batched(None, order.encode(), opA.encode(), opB.encode(), m, n, k,
                                       beta, ptrs[0], lda, sA, ptrs[1], ldb, sB, ptrs[2], ldc, sC,
                                       batch, None)
    return st, (lib.lrb_last_error(None) or b"").decode()


def test_validation_passes_then_needs_a_context():
    st, msg = _strided()
    assert st == _lib.LRB_ERR_ARG and "null ctx" in msg


@pytest.mark.parametrize("kw,status,text", [
    (dict(lda=3), _lib.LRB_ERR_SHAPE, "lda is 3 but A is 4x2"),
    (dict(ldb=1), _lib.LRB_ERR_SHAPE, "ldb is 1 but B is 2x3"),
    (dict(ldc=2), _lib.LRB_ERR_SHAPE, "ldc is 2 but C is 4x3"),
    (dict(sC=5), _lib.LRB_ERR_SHAPE, "items would overlap"),
    (dict(m=-1), _lib.LRB_ERR_SHAPE, "must be >= 0"),
    (dict(beta=0.5), _lib.LRB_ERR_UNSUPPORTED, "beta must be 0 or 1"),
    (dict(order="X"), _lib.LRB_ERR_ARG, "order"),
    (dict(opA="Q"), _lib.LRB_ERR_ARG, "opA"),
    (dict(ptrs=(0, 16, 16)), _lib.LRB_ERR_ARG, "null"),
    (dict(order="R", lda=1), _lib.LRB_ERR_SHAPE, "row-major"),
    (dict(m=2 ** 31), _lib.LRB_ERR_UNSUPPORTED, "2^31"),
])
def test_validation_errors(kw, status, text):
    st, msg = _strided(**kw)
    assert st == status, msg
    assert text in msg


def test_empty_and_degenerate_shapes_validate():
    # batch 0, m 0 and k 0 are legal (no-ops / zero fill), like the reference loops
    for kw in (dict(batch=0), dict(m=0, lda=1, ldc=1, sC=0), dict(k=0, lda=4, ldb=1)):
        st, msg = _strided(**kw)
        assert st == _lib.LRB_ERR_ARG and "null ctx" in msg, msg


# -------------------------------------------------- reference-shaped errors
def test_dense_gemm_naive_error_texts_match_reference():
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "shape_errors.json")))
    for c in cases:
        a, b, o = P.DenseBlock(*c["a"]), P.DenseBlock(*c["b"]), P.DenseBlock(*c["out"])
        with pytest.raises(P.ShapeError) as e:
            P.dense_gemm_naive(a, b, o)
        assert str(e.value) == c["error"]


def test_dense_block_mirror():
    b = P.DenseBlock.identity(3)
    assert b.at(1, 1) == 1.0 and b.at(0, 1) == 0.0
    with pytest.raises(P.ShapeError):
        P.DenseBlock(2, 2, [1.0, 2.0, 3.0])


def test_item_accounting():
    assert P.item_flops(256, 16, 256) == 2 * 256 * 16 * 256
    assert P.item_bytes(256, 16, 256) == 8 * (256 * 256 + 256 * 16 + 256 * 16)
    assert P.item_bytes(2, 2, 2, 1.0) == 8 * (4 + 4 + 8)


@pytest.mark.parametrize("args,status,text", [
    (dict(rank=0), _lib.LRB_ERR_SHAPE, "LowRankOperand: rank must be >= 1"),
    (dict(m=3), _lib.LRB_ERR_SHAPE, "need m >= rank and n >= rank, got (3, 8, 4)"),
    (dict(ldo=7), _lib.LRB_ERR_SHAPE, "ldo is 7 but out is 8x8"),
    (dict(so=10), _lib.LRB_ERR_SHAPE, "output items would overlap"),
    (dict(ptr=0), _lib.LRB_ERR_ARG, "null operand"),
    (dict(), _lib.LRB_ERR_ARG, "null ctx"),
])
def test_lowrank_expand_validation(args, status, text):
    # LowRankOperand's invariants and messages (low_rank.hpp:56-61), before any device work
    a = dict(batch=2, m=8, n=8, rank=4, ldo=8, so=64, ptr=16)
    a.update(args)
    p = a["ptr"]
    st = lib.lrb_lowrank_expand(None, a["batch"], a["m"], a["n"], a["rank"], 16, a["m"] * a["rank"],
                                16, 16, 16, 32, p, a["ldo"], a["so"], None)
    assert st == status
    assert text in (lib.lrb_last_error(None) or b"").decode()
