"""Host-timed probes of the widened rows (GPU box): BLR matvec eager / host-API
per call, low-rank r>32 eager vs graph. Prints one JSON line per probe."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2311_07602_b200 import Context  # noqa: E402
from paper_2311_07602_b200 import lowrank as L  # noqa: E402
from paper_2311_07602_b200 import workloads as W  # noqa: E402
from paper_2311_07602_b200.lrbatch import _check, lib  # noqa: E402


def wall(fn, reps, ctx):
    fn()
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    ctx.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def probe_blr(name):
    import bench_rows as R

    w = W.get_blr(name)
    ctx = Context(0)
    s = ctx.stream()
    m, rhs = R.blr_host(w)
    h = m.device_handle(ctx)
    d_rhs, d_y = ctx.to_device(rhs.data), ctx.empty(w.n * w.nrhs)
    y = np.zeros(w.n * w.nrhs)
    dev = lambda: _check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, w.nrhs, d_y.ptr,  # noqa
                                                    s.handle), ctx._h)
    host = lambda: _check(lib.lrb_blr_matvec(ctx._h, h, rhs.data.ctypes.data, w.nrhs,  # noqa
                                             y.ctypes.data), ctx._h)

    def dev_sync():
        dev()
        s.synchronize()

    out = {"probe": name, "device_eager_ms": wall(dev, 50, ctx),
           "device_eager_sync_ms": wall(dev_sync, 20, ctx), "host_api_ms": wall(host, 20, ctx)}
    with ctx.capture(s) as cap:
        dev()
    g = cap.graph
    out["device_graph_ms"] = wall(lambda: g.launch(s), 50, ctx)
    print(json.dumps(out), flush=True)
    ctx.close()


def probe_lowrank(name):
    w = W.get_lowrank(name)
    ctx = Context(0)
    s = ctx.stream()
    n, r, blk = w.batch, w.rank, w.block
    bufs = [ctx.empty(n * r * blk), ctx.empty(n * blk * r), ctx.empty(n * r * r),
            ctx.empty(n * r * r), ctx.empty(n * r * r)]
    for i, (rows, cols) in enumerate(((blk, r), (r, blk), (r, r), (r, r))):
        ctx.fill_uniform(bufs[i], rows, cols, rows, rows * cols, n, w.seed, i, 0)
    step = lambda: L.lowrank_multiply_device(ctx, n, blk, r, *bufs, stream=s)  # noqa: E731
    out = {"probe": name, "eager_ms": wall(step, 10, ctx)}
    with ctx.capture(s) as cap:
        step()
    g = cap.graph
    out["graph_ms"] = wall(lambda: g.launch(s), 10, ctx)
    out["gflops_graph"] = w.flops() / out["graph_ms"] / 1e6
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    for a in sys.argv[1:]:
        (probe_blr if a.startswith("blr_") else probe_lowrank)(a)
