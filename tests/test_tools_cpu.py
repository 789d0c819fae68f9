"""Host-side measurement tooling: the scripts that turn profiles/ into the
tables of DESIGN.md and summarise ncu output run on the committed files."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    return subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True,
                          timeout=120)


def test_design_tables_follow_the_committed_profiles():
    # --check prints the sweep and low-rank tables without touching DESIGN.md;
    # the rows it prints must be the ones the document carries
    r = _run(["tools/design_tables.py", "--check"])
    assert r.returncode == 0, r.stderr
    design = open(os.path.join(ROOT, "DESIGN.md")).read()
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith("| cfg") or ln.startswith("| r = ")]
    assert len(rows) >= 15
    for ln in rows:
        assert ln in design, ln[:80]


def test_rows_table_prints_every_widened_row():
    r = _run(["tools/rows_table.py", "profiles/bench_rows_r02.jsonl", "profiles/traffic.json"])
    assert r.returncode == 0, r.stderr
    names = {json.loads(ln)["config"]["workload"]
             for ln in open(os.path.join(ROOT, "profiles/bench_rows_r02.jsonl")) if ln.startswith("{")}
    for n in names:
        assert f"`{n}`" in r.stdout


def test_traffic_json_carries_pipe_evidence_for_every_config():
    # one ncu metrics pass: DRAM bytes, duration, DRAM % and DMMA-pipe % per kernel
    t = json.load(open(os.path.join(ROOT, "profiles/traffic.json")))
    for name in ["cfg1", "cfg2", "cfg4", "cfg5", "cfg3_b256_r32", "lr_r64_b2048",
                 "blr_n16384_b256_r16_k16", "lrx_m512_r8", "blrd_n16384_b512_r16"]:
        e = t[name]
        assert e["dram_bytes_per_launch"] > 0 and e["kernel_s"] > 0
        assert 0 < e["dram_pct"] <= 100 and 0 <= e["dmma_pct"] <= 100
    # and the launch list of the default bench command names the cfg4 kernel
    text = open(os.path.join(ROOT, "profiles/launches_r02.csv")).read()
    rows = list(csv.DictReader(text[text.find('"ID"'):].splitlines()))
    assert any("lrb_varn_kernel" in r["Kernel Name"] for r in rows)
