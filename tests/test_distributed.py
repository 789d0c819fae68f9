"""CPU, world_size 2 over gloo: the N>1 path of the harness.

The batch is independent per item, so multi-GPU is a shard plan plus a
barrier and a max-over-ranks of the device time — no data-path collective.
Each rank here computes its contiguous shard of a cfg5-shaped window with the
CPU oracle from GLOBAL item indices (the counter RNG), rank 0 gathers and checks
the result is bitwise the unsharded one, and the bench's reduction helpers
(max of times, sum of items) are exercised exactly as bench.py uses them.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch

    import bench
    import oracle as O
    from paper_2311_07602_b200 import workloads as W

    w_world, w_rank, w_local, pg = bench.dist_setup()
    assert (w_world, w_rank, w_local) == (world, rank, rank)
    # a 24-item window of cfg5 (512x512 * 512x32), items 1000..1023, shrunk k
    base, count = 1000, 24
    w = W.Strided("cfg5win", 64, 32, 64, count, seed=4)
    from paper_2311_07602_b200 import shard_plan

    b = shard_plan(count, world)
    lo, hi = b[rank], b[rank + 1]
    n = hi - lo
    A = O.fill_uniform(w.a_rows, w.a_cols, w.lda, w.sA, n, w.seed, W.ROLE_A, base + lo)
    B = O.fill_uniform(w.b_rows, w.b_cols, w.ldb, w.sB, n, w.seed, W.ROLE_B, base + lo)
    Cm = np.zeros(w.sC * n)
    O.dgemm_strided("C", "N", "N", w.m, w.n, w.k, 0.0, A, w.lda, w.sA, B, w.ldb, w.sB, Cm, w.ldc,
                    w.sC, n)
    # gather shards to rank 0
    parts = [torch.zeros(w.sC * (b[g + 1] - b[g]), dtype=torch.float64) for g in range(world)]
    mine = torch.from_numpy(Cm)
    if rank == 0:
        dist.gather(mine, gather_list=parts, dst=0)
    else:
        dist.gather(mine, dst=0)
    # the bench's reductions: max of per-rank device time, sum of items
    t = bench.all_max(pg, float(rank + 1) * 1.5)
    s = bench.all_sum(pg, float(n))
    bench.barrier(pg)
    if rank == 0:
        whole = torch.cat(parts).numpy()
        A = O.fill_uniform(w.a_rows, w.a_cols, w.lda, w.sA, count, w.seed, W.ROLE_A, base)
        B = O.fill_uniform(w.b_rows, w.b_cols, w.ldb, w.sB, count, w.seed, W.ROLE_B, base)
        ref = np.zeros(w.sC * count)
        O.dgemm_strided("C", "N", "N", w.m, w.n, w.k, 0.0, A, w.lda, w.sA, B, w.ldb, w.sB, ref,
                        w.ldc, w.sC, count)
        with open(os.path.join(out_dir, "result.txt"), "w") as f:
            f.write(f"{int(np.array_equal(whole, ref))} {t} {s}\n")
    dist.destroy_process_group()


def test_two_rank_shards_reassemble_bitwise(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    eq, t, s = open(tmp_path / "result.txt").read().split()
    assert eq == "1", "sharded result differs from the unsharded batch"
    assert float(t) == 3.0  # max over ranks
    assert float(s) == 24.0  # all items accounted once


def test_rank_items_partitions():
    import sys

    sys.path.insert(0, ROOT)
    import bench
    from paper_2311_07602_b200 import workloads as W

    w5 = W.get("cfg5")
    spans = [bench.rank_items(w5, 8, r) for r in range(8)]
    assert [s[1] for s in spans] == [16384] * 8 and spans[0][2] == "strong"
    assert sum(s[1] for s in spans) == w5.batch
    assert [s[0] for s in spans] == [r * 16384 for r in range(8)]
    w2 = W.get("cfg2")
    s2 = [bench.rank_items(w2, 4, r) for r in range(4)]
    assert all(s[1] == 4096 and s[2] == "weak" for s in s2)
    assert [s[0] for s in s2] == [0, 4096, 8192, 12288]
