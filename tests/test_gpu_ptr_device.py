"""GPU: pointer-array batches with DEVICE descriptor arrays
(lrb_dgemm_ptr_batched_device). The caller here is GPU-resident:
torch kernels build the cfg4 descriptor arrays (shapes and arena offsets by a
device cumsum) and the call runs without any host round trip, eagerly and
captured in a CUDA graph. Every item is checked bitwise against the oracle's
FMA chain; misaligned operands (the generic kernel), k = 0, row-major calls
and invalid descriptors (the device `info` pair) are covered too."""
import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _sync():
    torch.cuda.synchronize()


def _class_sample(w, per_class=2):
    """items covering every (b, r) class of cfg4, plus a contiguous run"""
    seen, items = {}, []
    for i in range(w.batch):
        key = (w.bs[i], w.rs[i])
        if seen.get(key, 0) < per_class:
            seen[key] = seen.get(key, 0) + 1
            items.append(i)
    return sorted(set(items) | set(range(64)))


def _device_descriptors(ctx, w, items):
    """arenas filled on device, descriptor arrays built on device by torch"""
    dev = torch.device("cuda", 0)
    b = torch.tensor([w.bs[i] for i in items], dtype=torch.int64, device=dev)
    r = torch.tensor([w.rs[i] for i in items], dtype=torch.int64, device=dev)

    def offsets(nbytes):  # 256-byte aligned exclusive cumsum, on the device
        al = (nbytes + 255) // 256 * 256
        return torch.cumsum(al, 0) - al, int(al.sum().item())

    oa, na = offsets(8 * b * b)
    ob, nb = offsets(8 * b * r)
    oc, nc = offsets(8 * b * r)
    arena = [ctx.malloc(na), ctx.malloc(nb), ctx.malloc(nc)]
    pa = oa + arena[0].ptr
    pb = ob + arena[1].ptr
    pc = oc + arena[2].ptr
    # inputs through the library's own generator (global item indices)
    hb, hr = [w.bs[i] for i in items], [w.rs[i] for i in items]
    pa_h, pb_h = pa.cpu().tolist(), pb.cpu().tolist()
    for j, i in enumerate(items):
        ctx.fill_uniform_ptr([pa_h[j]], [hb[j]], [hb[j]], [hb[j]], w.seed, W.ROLE_A, i)
        ctx.fill_uniform_ptr([pb_h[j]], [hb[j]], [hr[j]], [hb[j]], w.seed, W.ROLE_B, i)
    arena[2].fill_bytes(0xFF)  # NaN: beta = 0 must overwrite every entry
    ctx.synchronize()
    desc = dict(m=b, n=r, k=b.clone(), lda=b.clone(), ldb=b.clone(), ldc=b.clone(), A=pa, B=pb,
                C=pc)
    return desc, arena, pc.cpu().tolist()


def _call(ctx, desc, batch, beta=0.0, info=None, stream=None, order="C", opA="N", opB="N"):
    d = desc
    ctx.dgemm_ptr_batched_device(order, opA, opB, batch, d["m"].data_ptr(), d["n"].data_ptr(),
                                 d["k"].data_ptr(), d["A"].data_ptr(), d["lda"].data_ptr(),
                                 d["B"].data_ptr(), d["ldb"].data_ptr(), d["C"].data_ptr(),
                                 d["ldc"].data_ptr(), beta,
                                 info.data_ptr() if info is not None else None, stream)


def _check_cfg4(ctx, w, items, pc_h):
    import ctypes as C

    from paper_2311_07602_b200.lrbatch import _check, lib

    for j, i in enumerate(items):
        bb, rr = w.bs[i], w.rs[i]
        got = np.empty(bb * rr)
        _check(lib.lrb_memcpy_d2h(ctx._h, got.ctypes.data, C.c_void_p(pc_h[j]), got.nbytes), ctx._h)
        A = O.fill_uniform(bb, bb, bb, 0, 1, w.seed, W.ROLE_A, i)
        B = O.fill_uniform(bb, rr, bb, 0, 1, w.seed, W.ROLE_B, i)
        exp = np.zeros(bb * rr)
        O.dgemm_strided("C", "N", "N", bb, rr, bb, 0.0, A, bb, 0, B, bb, 0, exp, bb, 0, 1,
                        threads=8)
        assert np.array_equal(got, exp), f"cfg4 item {i} (b={bb}, r={rr})"


def test_cfg4_classes_device_built_descriptors(ctx):
    w = W.get("cfg4")
    items = _class_sample(w)
    desc, arena, pc_h = _device_descriptors(ctx, w, items)
    info = torch.full((2,), 7, dtype=torch.int64, device="cuda")
    _sync()
    _call(ctx, desc, len(items), info=info)
    ctx.synchronize()
    assert info.cpu().tolist() == [0, -1]
    _check_cfg4(ctx, w, items, pc_h)


def test_cfg4_device_descriptors_in_a_graph(ctx):
    w = W.get("cfg4")
    items = _class_sample(w, per_class=1)
    desc, arena, pc_h = _device_descriptors(ctx, w, items)
    _sync()
    s = ctx.stream()
    n0 = ctx.launch_count
    with ctx.capture(s) as cap:
        _call(ctx, desc, len(items), stream=s)
    assert ctx.launch_count == n0 and cap.graph.launches >= 7
    for _ in range(2):  # replays (the tile tickets reset at the end of each launch)
        arena[2].fill_bytes(0xFF)
        ctx.synchronize()
        cap.graph.launch(s)
        s.synchronize()
        _check_cfg4(ctx, w, items, pc_h)


class RaggedDevice:
    """ragged shapes with padded / odd leading dimensions and unaligned
    bases, descriptor arrays uploaded to the device"""

    def __init__(self, ctx, order, opA, opB, beta, seed, odd=True, dims=None):
        rng = np.random.default_rng(seed)
        self.ctx, self.order, self.opA, self.opB, self.beta = ctx, order, opA, opB, beta
        dims = dims or [(70, 9, 50), (130, 40, 17), (33, 64, 96), (256, 16, 256), (1, 1, 1),
                        (12, 7, 0), (65, 57, 129), (128, 64, 64), (200, 100, 33), (6, 3, 2)]
        self.dims = dims
        self.h = []
        ptrs = {"A": [], "B": [], "C": []}
        lds = {"lda": [], "ldb": [], "ldc": []}
        self.bufs = []
        for q, (m, n, k) in enumerate(dims):
            def st(op, r, c):
                return (c, r) if op == "T" else (r, c)
            sa, sb, sc = st(opA, m, k), st(opB, k, n), (m, n)
            def ld(shape, extra):
                return max(1, shape[1] if order == "R" else shape[0]) + extra
            pad = int(rng.integers(0, 3)) if odd else 0
            la, lb, lc = ld(sa, pad), ld(sb, pad), ld(sc, pad)
            def size(shape, l):
                r_, c_ = shape
                if r_ == 0 or c_ == 0:
                    return 1
                return (r_ - 1) * l + c_ if order == "R" else (c_ - 1) * l + r_
            off = int(rng.integers(0, 2)) if odd else 0  # 8-byte (not 16-byte) aligned bases
            a = rng.uniform(-1, 1, size(sa, la) + off)
            b = rng.uniform(-1, 1, size(sb, lb) + off)
            c = rng.uniform(-1, 1, size(sc, lc) + off) if beta else np.full(size(sc, lc) + off, np.nan)
            da, db, dc = ctx.to_device(a), ctx.to_device(b), ctx.to_device(c)
            self.bufs += [da, db, dc]
            self.h.append((a[off:], b[off:], c.copy(), off))
            ptrs["A"].append(da.ptr + 8 * off)
            ptrs["B"].append(db.ptr + 8 * off)
            ptrs["C"].append(dc.ptr + 8 * off)
            lds["lda"].append(la)
            lds["ldb"].append(lb)
            lds["ldc"].append(lc)
            self.dc = getattr(self, "dc", []) + [dc]
        t = lambda xs: torch.tensor(xs, dtype=torch.int64, device="cuda")  # noqa: E731
        self.desc = dict(m=t([d[0] for d in dims]), n=t([d[1] for d in dims]),
                         k=t([d[2] for d in dims]), A=t(ptrs["A"]), B=t(ptrs["B"]),
                         C=t(ptrs["C"]), **{kk: t(v) for kk, v in lds.items()})
        self.lds = lds

    def run(self, info=None):
        _sync()
        _call(self.ctx, self.desc, len(self.dims), beta=self.beta, info=info, order=self.order,
              opA=self.opA, opB=self.opB)
        self.ctx.synchronize()

    def check(self):
        ms = [d[0] for d in self.dims]
        ns = [d[1] for d in self.dims]
        ks = [d[2] for d in self.dims]
        A = [h[0] for h in self.h]
        B = [h[1] for h in self.h]
        exp = [h[2][h[3]:].copy() for h in self.h]
        O.dgemm_ptr(self.order, self.opA, self.opB, ms, ns, ks, A, self.lds["lda"], B,
                    self.lds["ldb"], exp, self.lds["ldc"], self.beta)
        for q, (dc, h, e) in enumerate(zip(self.dc, self.h, exp)):
            got = dc.download(h[2].size)[h[3]:]
            assert np.array_equal(got, e, equal_nan=True), f"item {q} {self.dims[q]}"


@pytest.mark.parametrize("order", ["C", "R"])
@pytest.mark.parametrize("ops", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_ragged_misaligned_all_ops(ctx, order, ops, beta):
    c = RaggedDevice(ctx, order, ops[0], ops[1], beta, seed=len(order) + ord(ops[0]) + 3 * int(beta))
    info = torch.zeros(2, dtype=torch.int64, device="cuda")
    c.run(info)
    assert info.cpu().tolist() == [0, -1]
    c.check()


@pytest.mark.parametrize("ops", [("N", "N"), ("T", "T")])
def test_aligned_shapes_single_launch_path(ctx, ops):
    c = RaggedDevice(ctx, "C", ops[0], ops[1], 0.0, seed=5, odd=False)
    c.run()
    c.check()


def test_invalid_descriptors_are_skipped_and_reported(ctx):
    c = RaggedDevice(ctx, "C", "N", "N", 0.0, seed=9, odd=False)
    lda = c.desc["lda"]
    lda[3] = 1  # too small for 256 rows
    c.desc["n"][6] = -1
    c.run(info=(info := torch.zeros(2, dtype=torch.int64, device="cuda")))
    assert info.cpu().tolist() == [2, 3]
    # the valid items are still computed (the skipped ones are untouched NaN)
    for q in (0, 1, 2, 4, 7, 8):
        m, n, k = c.dims[q]
        a, b, cc, off = c.h[q]
        exp = cc[off:].copy()
        O.dgemm_ptr("C", "N", "N", [m], [n], [k], [a], [c.lds["lda"][q]], [b], [c.lds["ldb"][q]],
                    [exp], [c.lds["ldc"][q]], 0.0)
        assert np.array_equal(c.dc[q].download(cc.size)[off:], exp, equal_nan=True)
    assert np.isnan(c.dc[3].download(c.h[3][2].size)).all()


def test_empty_batch(ctx):
    info = torch.full((2,), 5, dtype=torch.int64, device="cuda")
    _sync()
    ctx.dgemm_ptr_batched_device("C", "N", "N", 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0.0,
                                 info.data_ptr())
    ctx.synchronize()
    assert info.cpu().tolist() == [0, -1]


class SpanDevice(RaggedDevice):
    """aligned operands whose byte spans sit on either side of 128 KiB: the
    encoded tensor map carries a large-tensor flag tensormap.replace does not
    recompute (csrc/lrb_ptr_device.cu, MapTemplates)"""

    def __init__(self, ctx, opA, opB):
        self.DIMS = [(128, 8, 128), (126, 8, 128), (128, 8, 126), (130, 16, 126), (256, 63, 256),
                     (256, 64, 256), (254, 64, 258), (64, 16, 256), (64, 16, 254), (2, 8, 8192),
                     (2, 8, 8194), (1024, 8, 16), (1024, 9, 18), (16384, 8, 2), (6, 3, 2),
                     (70, 9, 50), (512, 24, 512)]
        super().__init__(ctx, "C", opA, opB, 0.0, seed=13, odd=False, dims=self.DIMS)


@pytest.mark.parametrize("ops", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
def test_device_built_maps_equal_the_host_encoding(ctx, ops, monkeypatch, capfd):
    """LRB_PTRDEV_VERIFY=1 copies the device-built plan back and compares every
    single-launch item's tensor maps with cuTensorMapEncodeTiled's own encoding
    (all 128 bytes), and the tile list with the host's"""
    monkeypatch.setenv("LRB_PTRDEV_VERIFY", "1")
    c = SpanDevice(ctx, ops[0], ops[1])
    c.run()
    err = capfd.readouterr().err
    lines = [ln for ln in err.splitlines() if "[ptrdev verify]" in ln]
    assert lines and lines[-1].endswith(" 0 differences"), "\n".join(lines[-12:])
    assert "single-launch items" in lines[0] and not lines[0].split(": ")[1].startswith("0 ")
    c.check()


def test_device_built_maps_cfg4_classes_verified(ctx, monkeypatch, capfd):
    monkeypatch.setenv("LRB_PTRDEV_VERIFY", "1")
    w = W.get("cfg4")
    items = _class_sample(w, per_class=1)
    desc, arena, pc_h = _device_descriptors(ctx, w, items)
    _sync()
    _call(ctx, desc, len(items))
    ctx.synchronize()
    err = capfd.readouterr().err
    lines = [ln for ln in err.splitlines() if "[ptrdev verify]" in ln]
    assert lines and lines[-1].endswith(" 0 differences"), "\n".join(lines[-12:])
    _check_cfg4(ctx, w, items, pc_h)
