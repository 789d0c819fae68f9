"""Compare the reference's CPU drivers on the GPU box's host (naive vs packed,
per machine plan) for the low-rank product and the BLR matvec."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import bench_rows as R  # noqa: E402
import oracle as O  # noqa: E402
from paper_2311_07602_b200 import workloads as W  # noqa: E402

threads = os.cpu_count() or 1
for name in sys.argv[1:]:
    if name.startswith("lr_"):
        w = W.get_lowrank(name)
        b = R.lowrank_inputs_host(w, 64 * threads)
        args = (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)
        for which, machine in ((0, None), (2, "epyc-7502"), (2, "skylake-x-6148"), (2, "a64fx")):
            t0 = time.perf_counter()
            O.ref_lowrank(which, b.batch_size, w.block, w.rank, *args, workers=threads,
                          machine=machine)
            dt = O.ref_last_seconds()
            print(json.dumps({"w": name, "which": which, "machine": machine, "threads": threads,
                              "gflops": round(w.item_flops() * b.batch_size / dt / 1e9, 2)}))
    else:
        w = W.get_blr(name)
        m, rhs = R.blr_host(w)
        diag, u, x, vt = m.packed_arrays()
        for which, machine in ((1, None), (0, "epyc-7502"), (0, "skylake-x-6148")):
            t0 = time.perf_counter()
            O.ref_blr_matvec(which, w.n, w.block, w.rank, diag, u, x, vt, rhs.data, w.nrhs,
                             workers=threads, machine=machine)
            dt = O.ref_last_seconds()
            print(json.dumps({"w": name, "which": which, "machine": machine, "threads": threads,
                              "gflops": round(w.flops() / dt / 1e9, 2)}))
