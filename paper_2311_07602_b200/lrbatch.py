"""Reference-shaped host API over liblrb.so.

Mirrors the names, argument meaning and error behaviour of the reference's hot
path so a caller of ``lrbatch`` can switch to the B200 path:

* ``gemm_naive_raw``   <- proj/include/lrbatch/dense.hpp:43-56
* ``DenseBlock``       <- proj/include/lrbatch/dense.hpp:13-37
* ``dense_gemm_naive`` <- proj/include/lrbatch/dense.hpp:58-77 (ShapeError text)
* ``ShapeError`` / ``CapacityError`` <- proj/include/lrbatch/common.hpp:19-27

plus the batched entry points of ``include/lrb.h`` (strided, pointer-array,
host-buffer), the selector and the shard planner. All compute runs on the GPU
through the C-ABI; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import lib


# --------------------------------------------------------------- exceptions
class LrbError(RuntimeError):
    status = -1


class ShapeError(LrbError, ValueError):
    """reference ShapeError (std::invalid_argument), common.hpp:19-22"""

    status = _lib.LRB_ERR_SHAPE


class CapacityError(LrbError):
    """reference CapacityError (std::runtime_error), common.hpp:24-27"""

    status = _lib.LRB_ERR_CAPACITY


class ArgError(LrbError, ValueError):
    status = _lib.LRB_ERR_ARG


class CudaError(LrbError):
    status = _lib.LRB_ERR_CUDA


class UnsupportedError(LrbError, ValueError):
    status = _lib.LRB_ERR_UNSUPPORTED


class NoDeviceError(LrbError):
    status = _lib.LRB_ERR_NO_DEVICE


class IoError(LrbError):
    """reference IoError (common.hpp:34-37)"""

    status = _lib.LRB_ERR_IO


class ParseError(LrbError):
    """reference ParseError (common.hpp:29-32)"""

    status = _lib.LRB_ERR_PARSE


_EXC = {
    _lib.LRB_ERR_SHAPE: ShapeError,
    _lib.LRB_ERR_CAPACITY: CapacityError,
    _lib.LRB_ERR_ARG: ArgError,
    _lib.LRB_ERR_CUDA: CudaError,
    _lib.LRB_ERR_UNSUPPORTED: UnsupportedError,
    _lib.LRB_ERR_NO_DEVICE: NoDeviceError,
    _lib.LRB_ERR_IO: IoError,
    _lib.LRB_ERR_PARSE: ParseError,
}


def _check(status: int, ctx_ptr=None) -> None:
    if status == _lib.LRB_OK:
        return
    msg = lib.lrb_last_error(ctx_ptr)
    text = msg.decode() if msg else f"lrb status {status}"
    raise _EXC.get(status, LrbError)(text)


def _b(ch: str) -> bytes:
    if not isinstance(ch, (str, bytes)) or len(ch) != 1:
        raise ArgError(f"expected a single character, got {ch!r}")
    return ch.encode() if isinstance(ch, str) else ch


def _ptr(x) -> Optional[int]:
    """device/host address of a DeviceBuffer, PinnedBuffer, numpy array or int"""
    if x is None:
        return None
    if isinstance(x, (DeviceBuffer, PinnedBuffer)):
        return x.ptr
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return int(x)


def _host_array(x, name: str, writable: bool = False) -> np.ndarray:
    if not isinstance(x, np.ndarray) or x.dtype != np.float64 or not x.flags.c_contiguous:
        raise ArgError(f"{name} must be a C-contiguous float64 numpy array")
    if writable and not x.flags.writeable:
        raise ArgError(f"{name} must be writable")
    return x


# ------------------------------------------------------------------ buffers
class DeviceBuffer:
    """Device allocation owned by a Context (cudaMalloc through the C-ABI)."""

    def __init__(self, ctx: "Context", nbytes: int):
        self.ctx = ctx
        self.nbytes = int(nbytes)
        p = C.c_void_p()
        _check(lib.lrb_malloc(ctx._h, self.nbytes, C.byref(p)), ctx._h)
        self.ptr = p.value or 0

    def free(self) -> None:
        if self.ptr and self.ctx._h:
            lib.lrb_free(self.ctx._h, self.ptr)
        self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def upload(self, host: np.ndarray, offset_bytes: int = 0) -> "DeviceBuffer":
        host = np.ascontiguousarray(host)
        if offset_bytes + host.nbytes > self.nbytes:
            raise ArgError("upload larger than the buffer")
        _check(lib.lrb_memcpy_h2d(self.ctx._h, self.ptr + offset_bytes, host.ctypes.data,
                                  host.nbytes), self.ctx._h)
        return self

    def download(self, count: Optional[int] = None, dtype=np.float64,
                 offset_bytes: int = 0) -> np.ndarray:
        itemsize = np.dtype(dtype).itemsize
        if count is None:
            count = (self.nbytes - offset_bytes) // itemsize
        out = np.empty(count, dtype=dtype)
        if out.nbytes + offset_bytes > self.nbytes:
            raise ArgError("download larger than the buffer")
        _check(lib.lrb_memcpy_d2h(self.ctx._h, out.ctypes.data, self.ptr + offset_bytes,
                                  out.nbytes), self.ctx._h)
        return out

    def fill_bytes(self, value: int = 0) -> None:
        _check(lib.lrb_memset(self.ctx._h, self.ptr, value, self.nbytes), self.ctx._h)


class PinnedBuffer:
    """Page-locked host allocation (cudaMallocHost) exposed as a float64 numpy view."""

    def __init__(self, ctx: "Context", count: int):
        self.ctx = ctx
        self.nbytes = int(count) * 8
        p = C.c_void_p()
        _check(lib.lrb_host_alloc(ctx._h, self.nbytes, C.byref(p)), ctx._h)
        self.ptr = p.value or 0
        if self.nbytes:
            buf = (C.c_double * int(count)).from_address(self.ptr)
            self.array = np.ctypeslib.as_array(buf)
        else:
            self.array = np.empty(0, dtype=np.float64)

    def free(self) -> None:
        if self.ptr and self.ctx._h:
            self.array = None
            lib.lrb_host_free(self.ctx._h, self.ptr)
        self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Stream:
    def __init__(self, ctx: "Context"):
        self.ctx = ctx
        p = C.c_void_p()
        _check(lib.lrb_stream_create(ctx._h, C.byref(p)), ctx._h)
        self.handle = p.value

    def synchronize(self) -> None:
        _check(lib.lrb_stream_sync(self.ctx._h, self.handle), self.ctx._h)

    def destroy(self) -> None:
        if self.handle and self.ctx._h:
            lib.lrb_stream_destroy(self.ctx._h, self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class Event:
    def __init__(self, ctx: "Context"):
        self.ctx = ctx
        p = C.c_void_p()
        _check(lib.lrb_event_create(ctx._h, C.byref(p)), ctx._h)
        self.handle = p.value

    def record(self, stream: Optional[Stream] = None) -> "Event":
        _check(lib.lrb_event_record(self.ctx._h, self.handle, stream.handle if stream else None),
               self.ctx._h)
        return self

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        _check(lib.lrb_event_elapsed_ms(self.ctx._h, self.handle, end.handle, C.byref(ms)),
               self.ctx._h)
        return float(ms.value)

    def destroy(self) -> None:
        if self.handle and self.ctx._h:
            lib.lrb_event_destroy(self.ctx._h, self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class Graph:
    """A captured sequence of lrb launches (CUDA graph), replayed with one call."""

    def __init__(self, ctx: "Context", handle: int):
        self.ctx = ctx
        self.handle = handle

    @property
    def launches(self) -> int:
        return int(lib.lrb_graph_launches(self.handle))

    def launch(self, stream: "Stream") -> None:
        _check(lib.lrb_graph_launch(self.ctx._h, self.handle, stream.handle), self.ctx._h)

    def destroy(self) -> None:
        if self.handle and self.ctx._h:
            lib.lrb_graph_destroy(self.ctx._h, self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class _Capture:
    def __init__(self, ctx: "Context", stream: "Stream"):
        self.ctx, self.stream, self.graph = ctx, stream, None

    def __enter__(self):
        _check(lib.lrb_graph_begin(self.ctx._h, self.stream.handle), self.ctx._h)
        return self

    def __exit__(self, exc_type, exc, tb):
        h = C.c_void_p()
        st = lib.lrb_graph_end(self.ctx._h, self.stream.handle, C.byref(h))
        if exc_type is None:
            _check(st, self.ctx._h)
            self.graph = Graph(self.ctx, h.value)
        return False


def _i64arr(xs, n: int, name: str):
    a = np.ascontiguousarray(np.asarray(xs, dtype=np.int64))
    if a.shape != (n,):
        raise ArgError(f"{name} must have length {n}")
    return a, a.ctypes.data_as(C.POINTER(C.c_int64))


def _ptrarr(xs, n: int, name: str):
    if len(xs) != n:
        raise ArgError(f"{name} must have length {n}")
    arr = (C.c_void_p * n)(*[_ptr(x) for x in xs])
    return arr


class PtrPlan:
    """Descriptor of a pointer-array / variable-size batch (lrb_ptr_plan)."""

    def __init__(self, ctx: "Context", handle: int, keep):
        self.ctx = ctx
        self.handle = handle
        self._keep = keep

    @property
    def launches(self) -> int:
        return int(lib.lrb_ptr_plan_launches(self.handle))

    def execute(self, stream: Optional[Stream] = None) -> None:
        _check(lib.lrb_ptr_plan_execute(self.ctx._h, self.handle,
                                        stream.handle if stream else None), self.ctx._h)

    def destroy(self) -> None:
        if self.handle and self.ctx._h:
            lib.lrb_ptr_plan_destroy(self.ctx._h, self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


# ------------------------------------------------------------------ context
class Context:
    """One lrb_ctx: a device, its streams and cached workspace."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.lrb_create(int(device), C.byref(h)), None)
        self._h = h.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.lrb_destroy(self._h)
        self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- properties
    @property
    def device(self) -> int:
        return int(lib.lrb_ctx_device(self._h))

    @property
    def sm_count(self) -> int:
        return int(lib.lrb_ctx_sm_count(self._h))

    @property
    def launch_count(self) -> int:
        return int(lib.lrb_launch_count(self._h))

    @property
    def last_variant(self) -> Optional[str]:
        """name of the kernel that served the last strided GEMM on this context"""
        v = int(lib.lrb_last_variant(self._h))
        return None if v < 0 else lib.lrb_variant_name(v).decode()

    def mem_info(self):
        f, t = C.c_size_t(), C.c_size_t()
        _check(lib.lrb_mem_info(self._h, C.byref(f), C.byref(t)), self._h)
        return int(f.value), int(t.value)

    # -- resources
    def malloc(self, nbytes: int) -> DeviceBuffer:
        return DeviceBuffer(self, nbytes)

    def empty(self, count: int) -> DeviceBuffer:
        return DeviceBuffer(self, int(count) * 8)

    def to_device(self, host: np.ndarray) -> DeviceBuffer:
        """float64 copy on the device; integer arrays (descriptor arrays for
        lrb_dgemm_ptr_batched_device) keep their dtype"""
        host = np.asarray(host)
        host = np.ascontiguousarray(host, dtype=None if host.dtype.kind in "iu" else np.float64)
        return DeviceBuffer(self, host.nbytes).upload(host)

    def pinned(self, count: int) -> PinnedBuffer:
        return PinnedBuffer(self, count)

    def stream(self) -> Stream:
        return Stream(self)

    def event(self) -> Event:
        return Event(self)

    def synchronize(self) -> None:
        _check(lib.lrb_device_sync(self._h), self._h)

    def capture(self, stream: Stream) -> _Capture:
        """``with ctx.capture(s) as cap: ...`` records the launches on ``s`` into
        ``cap.graph`` (a CUDA graph) instead of running them"""
        return _Capture(self, stream)

    def l2_flush(self, stream: Optional[Stream] = None) -> None:
        _check(lib.lrb_l2_flush(self._h, stream.handle if stream else None), self._h)

    def l2_evict(self, stream: Optional[Stream] = None) -> None:
        """clean eviction (reads 2x L2): a cold start without dirty write-backs"""
        _check(lib.lrb_l2_evict(self._h, stream.handle if stream else None), self._h)

    def set_variant_override(self, name: Optional[str]) -> None:
        v = -1 if name is None else variant_from_name(name)
        if name is not None and v < 0:
            raise ArgError(f"unknown kernel variant {name!r}; known: {variant_names()}")
        _check(lib.lrb_set_variant_override(self._h, v), self._h)

    def set_loader(self, mode: Optional[str]) -> None:
        """None/'auto', 'segment' (per-segment bulk copies) or 'tma' (tensor maps)"""
        m = {None: -1, "auto": -1, "segment": 0, "tma": 1}.get(mode)
        if m is None:
            raise ArgError(f"unknown loader {mode!r}")
        _check(lib.lrb_set_loader_override(self._h, m), self._h)

    # -- hot path
    def dgemm_strided_batched(self, order, opA, opB, m, n, k, beta, A, lda, strideA, B, ldb,
                              strideB, Cm, ldc, strideC, batch, stream: Optional[Stream] = None):
        _check(lib.lrb_dgemm_strided_batched(
            self._h, _b(order), _b(opA), _b(opB), m, n, k, float(beta), _ptr(A), lda, strideA,
            _ptr(B), ldb, strideB, _ptr(Cm), ldc, strideC, batch,
            stream.handle if stream else None), self._h)

    def dgemm_strided_batched_host(self, order, opA, opB, m, n, k, beta, A, lda, strideA, B, ldb,
                                   strideB, Cm, ldc, strideC, batch):
        _host_array(A, "A")
        _host_array(B, "B")
        _host_array(Cm, "C", writable=True)
        _check(lib.lrb_dgemm_strided_batched_host(
            self._h, _b(order), _b(opA), _b(opB), m, n, k, float(beta), _ptr(A), lda, strideA,
            _ptr(B), ldb, strideB, _ptr(Cm), ldc, strideC, batch), self._h)

    def ptr_plan(self, order, opA, opB, m, n, k, A, lda, B, ldb, Cs, ldc, beta) -> PtrPlan:
        batch = len(m)
        ma, mp = _i64arr(m, batch, "m")
        na, np_ = _i64arr(n, batch, "n")
        ka, kp = _i64arr(k, batch, "k")
        la, lp = _i64arr(lda, batch, "lda")
        lb, lbp = _i64arr(ldb, batch, "ldb")
        lc, lcp = _i64arr(ldc, batch, "ldc")
        pa, pb, pc = _ptrarr(A, batch, "A"), _ptrarr(B, batch, "B"), _ptrarr(Cs, batch, "C")
        h = C.c_void_p()
        _check(lib.lrb_ptr_plan_create(self._h, _b(order), _b(opA), _b(opB), batch, mp, np_, kp,
                                       pa, lp, pb, lbp, pc, lcp, float(beta), C.byref(h)), self._h)
        return PtrPlan(self, h.value, (ma, na, ka, la, lb, lc, pa, pb, pc))

    def dgemm_ptr_batched(self, order, opA, opB, m, n, k, A, lda, B, ldb, Cs, ldc, beta,
                          stream: Optional[Stream] = None) -> None:
        batch = len(m)
        ma, mp = _i64arr(m, batch, "m")
        na, np_ = _i64arr(n, batch, "n")
        ka, kp = _i64arr(k, batch, "k")
        la, lp = _i64arr(lda, batch, "lda")
        lb, lbp = _i64arr(ldb, batch, "ldb")
        lc, lcp = _i64arr(ldc, batch, "ldc")
        pa, pb, pc = _ptrarr(A, batch, "A"), _ptrarr(B, batch, "B"), _ptrarr(Cs, batch, "C")
        _check(lib.lrb_dgemm_ptr_batched(self._h, _b(order), _b(opA), _b(opB), batch, mp, np_, kp,
                                         pa, lp, pb, lbp, pc, lcp, float(beta),
                                         stream.handle if stream else None), self._h)
        del ma, na, ka, la, lb, lc

    def dgemm_ptr_batched_device(self, order, opA, opB, batch, m, n, k, A, lda, B, ldb, Cs, ldc,
                                 beta, info=None, stream: Optional[Stream] = None) -> None:
        """pointer-array batch whose descriptor arrays are DEVICE addresses
        (int64 m/n/k/ld arrays, pointer arrays as int64 device addresses);
        asynchronous on `stream`; `info` an optional device int64[2]"""
        _check(lib.lrb_dgemm_ptr_batched_device(
            self._h, _b(order), _b(opA), _b(opB), int(batch), _ptr(m), _ptr(n), _ptr(k), _ptr(A),
            _ptr(lda), _ptr(B), _ptr(ldb), _ptr(Cs), _ptr(ldc), float(beta), _ptr(info),
            stream.handle if stream else None), self._h)

    def dgemm_ptr_batched_host(self, order, opA, opB, m, n, k, A, lda, B, ldb, Cs, ldc,
                               beta) -> None:
        """pointer-array batch over HOST blocks (raw addresses or numpy arrays);
        synchronous, copies pipelined with the kernels"""
        batch = len(m)
        ma, mp = _i64arr(m, batch, "m")
        na, np_ = _i64arr(n, batch, "n")
        ka, kp = _i64arr(k, batch, "k")
        la, lp = _i64arr(lda, batch, "lda")
        lb, lbp = _i64arr(ldb, batch, "ldb")
        lc, lcp = _i64arr(ldc, batch, "ldc")
        pa, pb, pc = _ptrarr(A, batch, "A"), _ptrarr(B, batch, "B"), _ptrarr(Cs, batch, "C")
        _check(lib.lrb_dgemm_ptr_batched_host(self._h, _b(order), _b(opA), _b(opB), batch, mp,
                                              np_, kp, pa, lp, pb, lbp, pc, lcp, float(beta)),
               self._h)
        del ma, na, ka, la, lb, lc

    # -- synthetic inputs (include/lrb_rng.h)
    def fill_uniform(self, buf, rows, cols, ld, stride, batch, seed, role, item_offset=0,
                     stream: Optional[Stream] = None) -> None:
        _check(lib.lrb_fill_uniform(self._h, _ptr(buf), rows, cols, ld, stride, batch, seed, role,
                                    item_offset, stream.handle if stream else None), self._h)

    def fill_uniform_ptr(self, bufs, rows, cols, ld, seed, role, item_offset=0,
                         stream: Optional[Stream] = None) -> None:
        batch = len(bufs)
        pa = _ptrarr(bufs, batch, "dst")
        ra, rp = _i64arr(rows, batch, "rows")
        ca, cp = _i64arr(cols, batch, "cols")
        la, lp = _i64arr(ld, batch, "ld")
        _check(lib.lrb_fill_uniform_ptr(self._h, pa, rp, cp, lp, batch, seed, role, item_offset,
                                        stream.handle if stream else None), self._h)


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


# ------------------------------------------------- reference-shaped API
def gemm_naive_raw(a: np.ndarray, b: np.ndarray, c: np.ndarray, m: int, k: int, n: int,
                   accumulate: bool, flops: Optional[np.ndarray] = None,
                   ctx: Optional[Context] = None) -> None:
    """Drop-in for lrbatch::gemm_naive_raw (dense.hpp:43-56) on host buffers.

    Row-major a (m x k), b (k x n), c (m x n) as flat float64 arrays; c is
    written in place (accumulated into when ``accumulate``). ``flops``, when
    given, is a one-element uint64 array incremented by 2*m*n*k like the
    reference's ``uint64_t* flops``. Computed on the GPU.
    """
    ctx = ctx or default_context()
    _host_array(a, "a")
    _host_array(b, "b")
    _host_array(c, "c", writable=True)
    if a.size < m * k or b.size < k * n or c.size < m * n:
        raise ShapeError(f"gemm_naive_raw: buffers smaller than {m}x{k}, {k}x{n}, {m}x{n}")
    fl = C.c_uint64(int(flops[0]) if flops is not None else 0)
    _check(lib.lrb_gemm_naive_raw(ctx._h, _ptr(a), _ptr(b), _ptr(c), m, k, n,
                                  1 if accumulate else 0, C.byref(fl)), ctx._h)
    if flops is not None:
        flops[0] = fl.value


class DenseBlock:
    """Row-major dense block (reference DenseBlock, dense.hpp:13-37)."""

    def __init__(self, rows: int, cols: int, data: Optional[Sequence[float]] = None):
        self.rows = int(rows)
        self.cols = int(cols)
        if data is None:
            self.data = np.zeros(self.rows * self.cols, dtype=np.float64)
        else:
            self.data = np.ascontiguousarray(np.asarray(data, dtype=np.float64).ravel()).copy()
            if self.data.size != self.rows * self.cols:
                raise ShapeError(
                    f"DenseBlock: data length {self.data.size} != rows*cols {self.rows * self.cols}")

    def at(self, i: int, j: int) -> float:
        return float(self.data[i * self.cols + j])

    def set(self, i: int, j: int, v: float) -> None:
        self.data[i * self.cols + j] = v

    @staticmethod
    def identity(n: int) -> "DenseBlock":
        b = DenseBlock(n, n)
        b.data[:: n + 1] = 1.0
        return b

    def as_matrix(self) -> np.ndarray:
        return self.data.reshape(self.rows, self.cols)


def dense_gemm_naive(a: DenseBlock, b: DenseBlock, out: Optional[DenseBlock] = None,
                     accumulate: bool = False, flops: Optional[np.ndarray] = None,
                     ctx: Optional[Context] = None) -> DenseBlock:
    """Mirror of both dense_gemm_naive overloads (dense.hpp:58-77).

    With ``out`` the product is written (or accumulated) into it and ``out`` is
    returned; without, a new block is returned. Shape errors raise ShapeError
    with the reference's text.
    """
    if a.cols != b.rows:
        raise ShapeError(
            f"dense_gemm_naive: a is {a.rows}x{a.cols} but b is {b.rows}x{b.cols}")
    if out is None:
        out = DenseBlock(a.rows, b.cols)
        accumulate = False
    elif out.rows != a.rows or out.cols != b.cols:
        raise ShapeError(
            f"dense_gemm_naive: output is {out.rows}x{out.cols}, expected {a.rows}x{b.cols}")
    gemm_naive_raw(a.data, b.data, out.data, a.rows, a.cols, b.cols, accumulate, flops, ctx)
    return out


# ----------------------------------------------------- selector / planner
def variant_names():
    return [lib.lrb_variant_name(i).decode() for i in range(lib.lrb_variant_count())]


def variant_from_name(name: str) -> int:
    return int(lib.lrb_variant_from_name(name.encode()))


def select(order, opA, opB, m, n, k, batch, ctx: Optional[Context] = None) -> dict:
    """Per-shape kernel choice (plan.hpp:66-100 role); host-only when ctx is None."""
    s = _lib.lrb_selection()
    h = ctx._h if ctx else None
    _check(lib.lrb_select(h, _b(order), _b(opA), _b(opB), m, n, k, batch, C.byref(s)), h)
    return {
        "variant": s.variant, "name": s.name.decode(), "tile_m": s.tile_m, "tile_n": s.tile_n,
        "tile_k": s.tile_k, "stages": s.stages, "threads": s.threads,
        "ctas_per_sm": s.ctas_per_sm, "tiles": s.tiles, "grid": s.grid,
        "intensity": s.intensity, "fp64_bound": bool(s.fp64_bound),
    }


def shard_plan(batch: int, nparts: int, cost: Optional[Sequence[float]] = None):
    """Contiguous shard boundaries [begin_0=0, ..., begin_n=batch] (bench.hpp:69-75)."""
    out = (C.c_int64 * (nparts + 1))()
    if cost is None:
        cp = None
    else:
        carr = np.ascontiguousarray(np.asarray(cost, dtype=np.float64))
        if carr.shape != (batch,):
            raise ArgError("cost must have length batch")
        cp = carr.ctypes.data_as(C.POINTER(C.c_double))
    _check(lib.lrb_shard_plan(batch, cp, nparts, out), None)
    return [int(x) for x in out]


def item_flops(m: int, n: int, k: int) -> float:
    return float(lib.lrb_item_flops(m, n, k))


def item_bytes(m: int, n: int, k: int, beta: float = 0.0) -> float:
    return float(lib.lrb_item_bytes(m, n, k, beta))


def device_count() -> int:
    return int(lib.lrb_device_count())


def version() -> str:
    return lib.lrb_version().decode()
