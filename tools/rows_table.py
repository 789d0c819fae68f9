#!/usr/bin/env python3
"""Markdown rows of DESIGN.md §5.2 from a bench_rows jsonl (GPU arm + reference arm).

    python tools/rows_table.py profiles/bench_rows_r02.jsonl [profiles/traffic.json]
"""
import json
import sys


def main():
    rows = [json.loads(line) for line in open(sys.argv[1]) if line.startswith("{")]
    traffic = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else {}
    ref = {r["config"]["workload"]: r for r in rows if r.get("impl") == "reference"}
    print("| workload | kernel | GPU GFLOP/s | ms/step | bound, frac | DRAM/alg | e2e GFLOP/s (host API) "
          "| reference CPU (GFLOP/s, driver) |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        if r.get("impl") == "reference":
            continue
        name = r["config"]["workload"]
        roof = r["roofline"]
        bound = "fp64" if roof["bound"] == "tensor" else "hbm"
        tr = roof.get("traffic")
        ratio = f"{tr / roof['algorithmic']:.2f}" if tr and roof.get("algorithmic") else "—"
        e2e = (r.get("e2e") or {}).get("value")
        rr = ref.get(name)
        cpu = "—"
        if rr:
            cb = rr.get("cpu_baseline") or {}
            smp = cb.get("sample", "")
            drv = smp.split("), ")[1].split(" (")[0] if "), " in smp else cb.get("kind", "")
            cpu = f"{rr['value']:.1f} ({drv}, {cb.get('cores', '?')} thr)"
        print(f"| `{name}` | {roof.get('kernel', '')} | {r['value']:.0f} | {r['ms_per_step']:.4g} | "
              f"{bound} {roof['frac']:.2f} | {ratio} | {e2e if e2e is not None else '—'} | {cpu} |")


if __name__ == "__main__":
    main()
