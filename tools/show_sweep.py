#!/usr/bin/env python3
"""pretty-print tools/sweep.py JSON lines"""
import json
import sys

for f in sys.argv[1:]:
    print("==", f)
    for line in open(f):
        if not line.startswith("{"):
            print(line.rstrip()[:160])
            continue
        d = json.loads(line)
        print(f"{d['config']:16s} {d['variant']:10s} ms={d['ms']:8.3f} GF/s={d['gflops']:9.1f} "
              f"GB/s={d['gbs']:7.1f} I={d['intensity']:5.2f} {d.get('bound', ''):4s} "
              f"roof={d['roofline_frac']:.3f}")
