"""LRBATCH1 batch files (reference batch_io.hpp:11-77; tests/test_core.cpp:148-175):
round trips, interchange with the reference's own save_batch / load_batch,
error classes and texts, and (GPU) streaming a file straight into HBM."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import IoError, ParseError
from paper_2311_07602_b200 import lowrank as L


def _ref_load(path):
    hdr = (C.c_int64 * 4)()
    L_ = O.ref_lib()
    L_.ref_load_batch.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_char_p, C.c_size_t]
    err = C.create_string_buffer(256)
    rc = L_.ref_load_batch(path.encode(), C.addressof(hdr), None, None, None, None, err, 256)
    if rc:
        return None, err.value.decode()
    n, k, ra, rb = list(hdr)
    arrs = [np.zeros(n * ra * k), np.zeros(n * k * rb), np.zeros(n * ra * ra), np.zeros(n * rb * rb)]
    rc = L_.ref_load_batch(path.encode(), C.addressof(hdr), *[a.ctypes.data for a in arrs], err, 256)
    return (tuple(hdr), arrs), None


def test_round_trip(tmp_path):
    b = L.LowRankBatch.random(5, 24, 6, 77)
    p = str(tmp_path / "b.lrb")
    L.save_batch(b, p)
    assert os.path.getsize(p) == 8 + 32 + 8 * (2 * 5 * 6 * 24 + 2 * 5 * 36)
    c = L.load_batch(p)
    assert (c.batch_size, c.block_size, c.rank_a, c.rank_b) == (5, 24, 6, 6)
    for name in ("a_vt_batch", "b_u_batch", "a_x_batch", "b_x_batch"):
        assert np.array_equal(getattr(b, name), getattr(c, name))
    assert np.all(c.g_xy_batch == 0.0)  # results are not stored


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_interchange_with_the_reference(tmp_path):
    b = L.LowRankBatch.random(3, 17, 4, 5)
    ours = str(tmp_path / "ours.lrb")
    L.save_batch(b, ours)
    (hdr, arrs), err = _ref_load(ours)
    assert err is None and hdr == (3, 17, 4, 4)
    assert np.array_equal(arrs[0], b.a_vt_batch) and np.array_equal(arrs[3], b.b_x_batch)
    theirs = str(tmp_path / "theirs.lrb")
    O.ref_lib().ref_save_batch.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64] + [C.c_void_p] * 4
    assert O.ref_lib().ref_save_batch(theirs.encode(), 3, 17, 4, b.a_vt_batch.ctypes.data,
                                      b.b_u_batch.ctypes.data, b.a_x_batch.ctypes.data,
                                      b.b_x_batch.ctypes.data) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_errors_match_reference(tmp_path):
    bad = str(tmp_path / "bad.lrb")
    open(bad, "wb").write(b"NOTABATCH" + b"\0" * 64)
    with pytest.raises(ParseError) as e:
        L.load_batch(bad)
    assert str(e.value) == f"not a batch file (bad magic): {bad}"
    trunc = str(tmp_path / "trunc.lrb")
    b = L.LowRankBatch.random(2, 8, 2, 1)
    L.save_batch(b, trunc)
    data = open(trunc, "rb").read()
    open(trunc, "wb").write(data[:-8])
    with pytest.raises(ParseError) as e:
        L.load_batch(trunc)
    assert str(e.value) == f"truncated batch payload: {trunc}"
    open(trunc, "wb").write(data[:20])
    with pytest.raises(ParseError) as e:
        L.load_batch(trunc)
    assert str(e.value) == f"truncated batch header: {trunc}"
    missing = str(tmp_path / "nope" / "x.lrb")
    with pytest.raises(IoError) as e:
        L.load_batch(missing)
    assert str(e.value) == f"cannot open for reading: {missing}"
    if O.ref_available():  # the same texts from the reference itself
        for path in (bad, trunc, missing):
            _, err = _ref_load(path)
            try:
                L.load_batch(path)
            except (ParseError, IoError) as ours:
                assert str(ours) == err


@pytest.mark.gpu
def test_device_load_and_multiply(ctx, tmp_path):
    b = L.LowRankBatch.random(64, 256, 16, 9)
    p = str(tmp_path / "dev.lrb")
    L.save_batch(b, p)
    hdr, bufs, g = L.load_batch_device(ctx, p)
    assert hdr == (64, 256, 16, 16)
    assert np.array_equal(bufs[1].download(), b.b_u_batch)
    L.lowrank_multiply_device(ctx, 64, 256, 16, *bufs, g)
    ctx.synchronize()
    L.fused_multiply(b, ctx=ctx)
    assert np.array_equal(g.download(), b.g_xy_batch)
