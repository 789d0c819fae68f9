#!/usr/bin/env bash
# One GPU-box pass that regenerates the round's measurement artefacts into
# gpurun_out/ (copied to profiles/ by hand after review):
#   gpurun -- 'bash tools/measure_round.sh r01'
# Every ncu command runs only after the same command exited 0 without ncu.
set -u
R=${1:-r01}
O=gpurun_out
mkdir -p $O
log() { echo "[measure] $*"; }

log "gpu tests"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests_gpu_$R.log 2>&1
log "tests rc=$? $(tail -1 $O/tests_gpu_$R.log)"

log "sweeps"
timeout 900 python tools/sweep.py > $O/sweep_$R.jsonl 2> $O/sweep_$R.err
log "sweep rc=$?"
timeout 600 python tools/sweep.py --configs cfg3r_b128_r8,cfg3r_b256_r16,cfg3r_b512_r32,cfg3r_b1024_r64,cfg3r_b2048_r16 > $O/sweep_${R}_rowmajor.jsonl 2>> $O/sweep_$R.err
log "sweep rowmajor rc=$?"
timeout 900 python tools/sweep_lowrank.py > $O/sweep_lowrank_$R.jsonl 2>> $O/sweep_$R.err
log "sweep lowrank rc=$?"

log "traffic pass"
if timeout 900 python tools/profile_all.py > $O/profile_order_plain.log 2>&1; then
  timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file $O/traffic_$R.csv python tools/profile_all.py \
    > $O/profile_order.log 2>&1
  log "ncu traffic rc=$?"
  python tools/ncu_summary.py traffic $O/traffic_$R.csv $O/profile_order.log $O/traffic.json
else
  log "profile_all failed: $(tail -3 $O/profile_order_plain.log)"
fi

log "bench"
if timeout 900 python bench.py > $O/bench_$R.json 2> $O/bench_$R.err; then
  cat $O/bench_$R.json
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_$R.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 \
    > $O/launches_$R.log 2>&1
  log "launch list rc=$?"
fi
timeout 900 python bench.py --impl reference > $O/bench_reference_$R.json 2>> $O/bench_$R.err
log "reference arm rc=$?"

log "full capture of the cfg2 kernel"
if timeout 300 python tools/profile_one.py --config cfg2 --launches 2 > /dev/null 2>&1; then
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"lrb_(gemm|panel)_kernel" \
    -c 1 -f -o $O/ncu_cfg2_$R python tools/profile_one.py --config cfg2 --launches 2 \
    > $O/ncu_cfg2_$R.log 2>&1
  log "ncu full rc=$?"
fi
log "done"
