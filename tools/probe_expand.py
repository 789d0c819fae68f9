#!/usr/bin/env python3
"""Write-streaming probe for the expansion kernel: the same ~8 GiB of output
in items of different shapes (contiguous row runs of n * 8 bytes), rank 8 /
16, each timed over several launches with CUDA events (one JSON line each).

    python tools/probe_expand.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2311_07602_b200 import Context  # noqa: E402
from paper_2311_07602_b200 import blr as B  # noqa: E402

OUT_BYTES = 8 << 30


def main():
    ctx = Context(0)
    s = ctx.stream()
    shapes = [(512, 512), (512, 256), (256, 1024), (1024, 256), (64, 4096), (128, 2048)]
    for r in (8, 16):
        for m, n in shapes:
            batch = OUT_BYTES // (8 * m * n)
            u, x, vt = ctx.empty(batch * m * r), ctx.empty(batch * r * r), ctx.empty(batch * r * n)
            for b_ in (u, x, vt):
                b_.fill_bytes(0)
            out = ctx.empty(batch * m * n)
            for env in ("1", "0"):
                os.environ["LRB_EXPAND_STREAM"] = env
                B.lowrank_expand_device(ctx, batch, m, n, r, u, x, vt, out, stream=s)
                s.synchronize()
                e0, e1 = ctx.event(), ctx.event()
                reps = 5
                e0.record(s)
                for _ in range(reps):
                    B.lowrank_expand_device(ctx, batch, m, n, r, u, x, vt, out, stream=s)
                e1.record(s)
                s.synchronize()
                ms = e0.elapsed_ms(e1) / reps
                byts = 8.0 * batch * (m * n + m * r + r * r + r * n)
                print(json.dumps({"m": m, "n": n, "r": r, "batch": batch,
                                  "form": "stream" if env == "1" else "two_gemms",
                                  "ms": round(ms, 4), "tbs": round(byts / ms / 1e9, 3)}),
                      flush=True)
            del u, x, vt, out
    os.environ.pop("LRB_EXPAND_STREAM", None)


if __name__ == "__main__":
    main()
