#!/usr/bin/env python3
"""Summarise ncu outputs for profiles/.

    python tools/ncu_summary.py rep  <file.ncu-rep>          # key metrics + stall reasons
    python tools/ncu_summary.py traffic <metrics.csv> <order.log> <out.json>
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.per_cycle_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic",
]


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h.split("stalled_")[1].split("_per_issue")[0]))
                except ValueError:
                    pass
        d["top_stalls_per_issue"] = [[n, round(v, 3)] for v, n in sorted(stalls, reverse=True)[:6]]
        out.append(d)
    print(json.dumps(out, indent=1))


def traffic(csv_path, order_path, out_path):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = {}
    for r in rows:
        kn = r["Kernel Name"]
        if "fill_" in kn or not ("lrb_" in kn or "blr_" in kn):
            continue
        key = int(r["ID"])
        per.setdefault(key, {"kernel": r["Kernel Name"][:120]})
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                 "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(unit, 1)
        per[key][r["Metric Name"]] = val * scale
    launches = [per[k] for k in sorted(per)]
    order = []
    items = {}
    for line in open(order_path):
        if "launches=" in line:
            name = line.split()[0]
            n = int(line.split("launches=")[1].split()[0])
            order += [name] * n
            if "items=" in line:
                items[name] = int(line.split("items=")[1].split()[0])
    res = {}
    for name, d in zip(order, launches):
        e = res.setdefault(name, {"launches": 0, "dram_bytes_per_launch": 0.0, "kernel_s": 0.0,
                                  "kernels": []})
        e["launches"] += 1
        e["dram_bytes_per_launch"] += d.get("dram__bytes_read.sum", 0) + d.get(
            "dram__bytes_write.sum", 0)
        t = d.get("gpu__time_duration.sum", 0)
        e["kernel_s"] += t
        e["kernels"].append(d["kernel"])
        # duration-weighted pipe evidence (present when the pass asked for it)
        for key, out in (("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
                         ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg."
                          "pct_of_peak_sustained_active", "dmma_pct")):
            if key in d:
                e[out + "_x_s"] = e.get(out + "_x_s", 0.0) + d[key] * t
    for name, e in res.items():  # a cfg4 "launch" is the plan's whole group set
        for out in ("dram_pct", "dmma_pct"):
            if out + "_x_s" in e:
                e[out] = round(e.pop(out + "_x_s") / e["kernel_s"], 2) if e["kernel_s"] else None
        e["note"] = "ncu serialised, cold-cache replay; bytes summed over the config's launches"
        if name in items:
            e["items"] = items[name]  # items per launch of the capture (bench scales by it)
    json.dump(res, open(out_path, "w"), indent=1)
    print(f"wrote {out_path}: {len(res)} configs from {len(launches)} launches")


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        rep(sys.argv[2])
    else:
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
