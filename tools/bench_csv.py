#!/usr/bin/env python3
"""The reference's `lrbatch bench` CSV (bench.hpp:125-230) from the GPU run_bench,
with the reference binary's naive_multiply_batch as the baseline column.

    python tools/bench_csv.py [--ranks 8,16,32] [--blocks 512,1024,2048] [--batch 10000]
                              [--reps 5] [--workers N] [--output profiles/bench_csv_r01.csv]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2311_07602_b200 import Context  # noqa: E402
from paper_2311_07602_b200 import bench_csv as BC  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="8,16,32")
    ap.add_argument("--blocks", default="512,1024,2048")
    ap.add_argument("--batch", type=int, default=10000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--output", default="")
    args = ap.parse_args()
    ctx = Context(0)

    def naive(batch, workers):
        O.ref_lowrank(0, batch.batch_size, batch.block_size, batch.rank_a, batch.a_vt_batch,
                      batch.b_u_batch, batch.a_x_batch, batch.b_x_batch, workers=workers)
        return O.ref_last_seconds()  # the driver alone

    rows = []
    for r in map(int, args.ranks.split(",")):
        for b in map(int, args.blocks.split(",")):
            cfg = BC.BenchConfig(batch_size=args.batch, block_size=b, rank=r,
                                 workers=args.workers, repetitions=args.reps, warmup_reps=1)
            rows.append(BC.run_bench(cfg, ctx=ctx, baseline=naive if O.ref_available() else None))
            print(BC.bench_csv_row(rows[-1]), file=sys.stderr, flush=True)
    print(BC.write_csv(rows, args.output), end="")


if __name__ == "__main__":
    main()
