"""BASELINE.json workloads as seeded synthetic batches.

There is no public dataset for this path: the reference and BASELINE.json
specify i.i.d. uniform[-1,1) entries per config seed, column-major, packed.
Inputs are generated ON THE DEVICE with the counter RNG of include/lrb_rng.h
(keyed by seed, role, GLOBAL item index and element), so every shard and
chunk regenerates exactly its slice and the host oracle can regenerate any
sampled item bit-for-bit.

Per-item accounting (beta = 0): flops 2mnk, algorithmic bytes 8(mk+kn+mn).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

ROLE_A, ROLE_B, ROLE_C, ROLE_SHAPE_B, ROLE_SHAPE_R = 0, 1, 2, 3, 4
GIB = 1 << 30

# ------------------------------------------------------------------ RNG (host)
_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_ROLE_MUL = 0xD1B54A32D192ED03
_ROLE_ADD = 0x632BE59BD9B4E019


def mix64(z: int) -> int:
    z &= _M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    z ^= z >> 31
    return z


def stream_key(seed: int, role: int) -> int:
    return mix64((seed * _GOLDEN + role * _ROLE_MUL + _ROLE_ADD) & _M64)


def bits(key: int, item: int, elem: int) -> int:
    return mix64((key + (((item << 32) | (elem & 0xFFFFFFFF)) & _M64) * _GOLDEN) & _M64)


def below(key: int, item: int, n: int) -> int:
    """lrb_below: uniform integer in [0, n) (include/lrb_rng.h)"""
    return ((bits(key, item, 0) >> 32) * n) >> 32


def uniform(key: int, item: int, elem: int) -> float:
    return (bits(key, item, elem) >> 11) * (1.0 / 4503599627370496.0) - 1.0


# ---------------------------------------------------------------- workloads
@dataclass
class Strided:
    """fixed-stride column-major batch: C_i = op(A_i) op(B_i)"""

    name: str
    m: int
    n: int
    k: int
    batch: int
    seed: int
    opA: str = "N"
    opB: str = "N"
    order: str = "C"
    beta: float = 0.0

    # (rows, cols) of each stored operand in the caller's order
    def _stored_a(self):
        return (self.k, self.m) if self.opA == "T" else (self.m, self.k)

    def _stored_b(self):
        return (self.n, self.k) if self.opB == "T" else (self.k, self.n)

    def _view(self, rc):
        """column-major view of a stored matrix: row-major r x c == column-major c x r"""
        return rc if self.order == "C" else (rc[1], rc[0])

    # the properties below describe the COLUMN-MAJOR VIEW of each buffer
    # (what lrb_fill_uniform fills); ld is the same number in either order
    @property
    def a_rows(self):
        return self._view(self._stored_a())[0]

    @property
    def a_cols(self):
        return self._view(self._stored_a())[1]

    @property
    def b_rows(self):
        return self._view(self._stored_b())[0]

    @property
    def b_cols(self):
        return self._view(self._stored_b())[1]

    @property
    def lda(self):
        return self.a_rows

    @property
    def ldb(self):
        return self.b_rows

    @property
    def ldc(self):
        return self.m if self.order == "C" else self.n

    @property
    def sA(self):
        return self.a_rows * self.a_cols

    @property
    def sB(self):
        return self.b_rows * self.b_cols

    @property
    def sC(self):
        return self.m * self.n

    def item_flops(self) -> float:
        return 2.0 * self.m * self.n * self.k

    def item_bytes(self) -> float:
        return 8.0 * (self.m * self.k + self.k * self.n + self.m * self.n)

    def flops(self, items: Optional[int] = None) -> float:
        return self.item_flops() * (self.batch if items is None else items)

    def bytes(self, items: Optional[int] = None) -> float:
        return self.item_bytes() * (self.batch if items is None else items)

    def describe(self) -> dict:
        return {"workload": self.name, "m": self.m, "n": self.n, "k": self.k,
                "batch": self.batch, "opA": self.opA, "opB": self.opB, "order": self.order,
                "seed": self.seed, "layout": "column-major, packed (stride = rows*cols)"}


@dataclass
class Variable:
    """pointer-array batch: C_i = A_i (b_i x b_i) B_i (b_i x r_i), 256-B aligned bases"""

    name: str
    batch: int
    seed: int
    b_choices: tuple = (256, 512, 1024)
    r_lo: int = 8
    r_hi: int = 64
    bs: List[int] = field(default_factory=list)
    rs: List[int] = field(default_factory=list)

    def __post_init__(self):
        kb = stream_key(self.seed, ROLE_SHAPE_B)
        kr = stream_key(self.seed, ROLE_SHAPE_R)
        nr = self.r_hi - self.r_lo + 1
        self.bs = [self.b_choices[below(kb, i, len(self.b_choices))] for i in range(self.batch)]
        self.rs = [self.r_lo + below(kr, i, nr) for i in range(self.batch)]

    def item_flops(self, i: int) -> float:
        b, r = self.bs[i], self.rs[i]
        return 2.0 * b * r * b

    def item_bytes(self, i: int) -> float:
        b, r = self.bs[i], self.rs[i]
        return 8.0 * (b * b + b * r + b * r)

    def flops(self, items=None) -> float:
        ids = range(self.batch) if items is None else items
        return sum(self.item_flops(i) for i in ids)

    def bytes(self, items=None) -> float:
        ids = range(self.batch) if items is None else items
        return sum(self.item_bytes(i) for i in ids)

    def describe(self) -> dict:
        return {"workload": self.name, "batch": self.batch, "seed": self.seed,
                "b": list(self.b_choices), "r": [self.r_lo, self.r_hi],
                "layout": "column-major, pointer array, 256-B aligned independent bases"}


def cfg3_batch(b: int, r: int, budget: int = 16 * GIB) -> int:
    """items whose A + B + C total ~16 GiB (BASELINE cfg3)"""
    return budget // (8 * (b * b + 2 * b * r))


CFG3_B = (128, 256, 512, 1024, 2048)
CFG3_R = (8, 16, 32, 64)


def get(name: str):
    """cfg1 | cfg2 | cfg3_b{B}_r{R} | cfg4 | cfg5"""
    if name == "cfg1":
        return Strided("cfg1", 256, 16, 256, 256, seed=0)
    if name == "cfg2":
        # low-rank expansion C = U V^T, U and V 512 x 32 column-major
        return Strided("cfg2", 512, 512, 32, 4096, seed=1, opA="N", opB="T")
    if name.startswith("cfg3"):
        # cfg3_b{B}_r{R}: BASELINE's column-major sweep; cfg3r_...: the same
        # shapes in the reference's own row-major storage (the drop-in case)
        parts = dict(p[0:1] and (p[0], p[1:]) for p in name.split("_")[1:])
        b, r = int(parts["b"]), int(parts["r"])
        order = "R" if name.startswith("cfg3r") else "C"
        return Strided(name, b, r, b, cfg3_batch(b, r), seed=2, order=order)
    if name == "cfg4":
        return Variable("cfg4", 8192, seed=3)
    if name == "cfg5":
        return Strided("cfg5", 512, 32, 512, 131072, seed=4)
    if name.startswith("lr_"):
        return get_lowrank(name)
    if name.startswith("blr_"):
        return get_blr(name)
    if name.startswith("lrx_"):
        return get_expand(name)
    if name.startswith("blrd_"):
        return get_blr_dense(name)
    raise KeyError(name)


def all_names() -> List[str]:
    return (["cfg1", "cfg2"] + [f"cfg3_b{b}_r{r}" for b in CFG3_B for r in CFG3_R]
            + ["cfg4", "cfg5"])


def align256(x: int) -> int:
    return (x + 255) // 256 * 256


def variable_layout(w: Variable, items: List[int]):
    """byte offsets of A_i, B_i, C_i inside three arenas, each base 256-B aligned"""
    oa = ob = oc = 0
    offs = []
    for i in items:
        b, r = w.bs[i], w.rs[i]
        offs.append((oa, ob, oc))
        oa = align256(oa + 8 * b * b)
        ob = align256(ob + 8 * b * r)
        oc = align256(oc + 8 * b * r)
    return offs, (oa, ob, oc)


@dataclass
class LowRank:
    """The paper's batched low-rank product over a LowRankBatch (row-major
    roles): G = A_X (A_Vt B_U) B_X, paper Section 6 shapes (batch 20000)."""

    name: str
    batch: int
    block: int
    rank: int
    seed: int = 7

    def item_flops(self) -> float:  # reference flops_per_item (low_rank.hpp:66-68)
        r, b = self.rank, self.block
        return 4.0 * r ** 3 + 2.0 * r * r * b

    def item_bytes(self) -> float:  # A_Vt, B_U, A_X, B_X read + G written
        r, b = self.rank, self.block
        return 8.0 * (2 * r * b + 3 * r * r)

    def flops(self, items=None) -> float:
        return self.item_flops() * (self.batch if items is None else items)

    def bytes(self, items=None) -> float:
        return self.item_bytes() * (self.batch if items is None else items)

    def describe(self) -> dict:
        return {"workload": self.name, "batch": self.batch, "block": self.block,
                "rank": self.rank, "seed": self.seed,
                "layout": "LowRankBatch: row-major roles packed contiguously"}


LOWRANK_R = (8, 16, 32, 64, 96, 128)
LOWRANK_B = (512, 1024, 2048)


def get_lowrank(name: str) -> LowRank:
    """lr_r{R}_b{B}[_n{batch}]"""
    parts = dict((p[0], p[1:]) for p in name.split("_")[1:])
    return LowRank(name, int(parts.get("n", 20000)), int(parts["b"]), int(parts["r"]))


@dataclass
class Blr:
    """BLR multi-RHS matvec y = M rhs (reference blr.hpp:141-175): n = tiles *
    block, dense diagonal tiles, rank-`rank` off-diagonal tiles, nrhs columns."""

    name: str
    n: int
    block: int
    rank: int
    nrhs: int
    seed: int = 11

    @property
    def tiles(self) -> int:
        return self.n // self.block

    def flops(self) -> float:
        T, b, r, k = self.tiles, self.block, self.rank, self.nrhs
        return T * 2.0 * b * b * k + T * (T - 1) * (4.0 * r * b * k + 2.0 * r * r * k)

    def bytes(self) -> float:
        T, b, r, k = self.tiles, self.block, self.rank, self.nrhs
        return 8.0 * (T * b * b + T * (T - 1) * (2 * b * r + r * r) + 2 * self.n * k)

    def describe(self) -> dict:
        return {"workload": self.name, "n": self.n, "block": self.block, "rank": self.rank,
                "nrhs": self.nrhs, "tiles": self.tiles, "seed": self.seed,
                "layout": "BlrMatrix tiles (row-major), rhs/y row-major n x nrhs"}


def get_blr(name: str) -> Blr:
    """blr_n{N}_b{B}_r{R}_k{nrhs}"""
    parts = dict((p[0], p[1:]) for p in name.split("_")[1:])
    return Blr(name, int(parts["n"]), int(parts["b"]), int(parts["r"]), int(parts["k"]))


@dataclass
class LrExpand:
    """Low-rank expansion out_i = (U_i X_i) Vt_i of `batch` m x m
    LowRankOperands of rank r (the per-tile expansion of reconstruct_dense,
    blr.hpp:75-78), all row-major and packed."""

    name: str
    batch: int
    m: int
    rank: int
    seed: int = 13

    def item_flops(self) -> float:  # UX: 2 m r^2, (UX) Vt: 2 m^2 r
        m, r = self.m, self.rank
        return 2.0 * m * r * r + 2.0 * m * m * r

    def item_bytes(self) -> float:  # U, X, Vt read, out written
        m, r = self.m, self.rank
        return 8.0 * (2 * m * r + r * r + m * m)

    def flops(self, items=None) -> float:
        return self.item_flops() * (self.batch if items is None else items)

    def bytes(self, items=None) -> float:
        return self.item_bytes() * (self.batch if items is None else items)

    def describe(self) -> dict:
        return {"workload": self.name, "batch": self.batch, "m": self.m, "n": self.m,
                "rank": self.rank, "seed": self.seed,
                "layout": "LowRankOperand roles row-major, packed; out m x m per item"}


def get_expand(name: str) -> LrExpand:
    """lrx_m{M}_r{R}[_b{batch}] (default batch: 8 GiB of output, like cfg2)"""
    parts = dict((p[0], p[1:]) for p in name.split("_")[1:])
    m = int(parts["m"])
    return LrExpand(name, int(parts.get("b", max(1, (8 << 30) // (8 * m * m)))), m,
                    int(parts["r"]))


@dataclass
class BlrDense:
    """BlrMatrix::reconstruct_dense (blr.hpp:62-86): the n x n dense matrix."""

    name: str
    n: int
    block: int
    rank: int
    seed: int = 11

    @property
    def tiles(self) -> int:
        return self.n // self.block

    def flops(self) -> float:
        T, b, r = self.tiles, self.block, self.rank
        return T * (T - 1) * (2.0 * b * r * r + 2.0 * b * b * r)

    def bytes(self) -> float:  # diag + factors read, n^2 written
        T, b, r = self.tiles, self.block, self.rank
        return 8.0 * (T * b * b + T * (T - 1) * (2 * b * r + r * r) + self.n * self.n)

    def describe(self) -> dict:
        return {"workload": self.name, "n": self.n, "block": self.block, "rank": self.rank,
                "tiles": self.tiles, "seed": self.seed,
                "layout": "BlrMatrix tiles in; n x n row-major out"}


def get_blr_dense(name: str) -> BlrDense:
    """blrd_n{N}_b{B}_r{R}"""
    parts = dict((p[0], p[1:]) for p in name.split("_")[1:])
    return BlrDense(name, int(parts["n"]), int(parts["b"]), int(parts["r"]))
