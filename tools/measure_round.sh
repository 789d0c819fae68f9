#!/usr/bin/env bash
# One GPU-box pass that regenerates the round's measurement artefacts into
# gpurun_out/ (copied to profiles/ by hand after review):
#   gpurun -- 'bash tools/measure_round.sh r02'
# Every ncu command runs only after the same command exited 0 without ncu.
set -u
R=${1:-r02}
O=gpurun_out
mkdir -p $O
log() { echo "[measure] $*"; }

log "gpu tests"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests_gpu_$R.log 2>&1
log "tests rc=$? $(tail -1 $O/tests_gpu_$R.log)"

log "bench lines (default cfg4, then every BASELINE config)"
timeout 900 python bench.py > $O/bench_$R.json 2> $O/bench_$R.err
log "bench rc=$? $(head -c 300 $O/bench_$R.json)"
timeout 900 python bench.py --impl reference > $O/bench_reference_$R.json 2>> $O/bench_$R.err
log "reference arm rc=$?"
for c in cfg1 cfg2 cfg5; do
  timeout 900 python bench.py --config $c > $O/bench_${c}_$R.json 2>> $O/bench_$R.err
  log "bench $c rc=$?"
done

log "probes (microbenchmarks only where their binaries were built: nvcc -arch=sm_100a -O3 -lcuda)"
timeout 600 python tools/probe_varn.py > $O/probe_varn_$R.jsonl 2>> $O/probe_$R.err
timeout 600 python tools/probe_cold.py > $O/probe_cold_$R.jsonl 2>> $O/probe_$R.err
[ -x tools/microbench/fp64_mix ] && timeout 300 ./tools/microbench/fp64_mix > $O/fp64_mix_$R.jsonl 2>> $O/probe_$R.err
[ -x tools/microbench/write_bw ] && timeout 300 ./tools/microbench/write_bw > $O/write_bw_$R.jsonl 2>> $O/probe_$R.err
[ -x tools/microbench/tmap_probe ] && timeout 120 ./tools/microbench/tmap_probe > $O/tmap_probe_$R.txt 2>> $O/probe_$R.err

log "widened rows, both arms"
bash tools/bench_rows_all.sh $R

log "sweeps"
timeout 900 python tools/sweep.py > $O/sweep_$R.jsonl 2> $O/sweep_$R.err
log "sweep rc=$?"
timeout 900 python tools/sweep_lowrank.py > $O/sweep_lowrank_$R.jsonl 2>> $O/sweep_$R.err
log "sweep lowrank rc=$?"

log "traffic pass"
if timeout 900 python tools/profile_all.py > $O/profile_order_plain.log 2>&1; then
  timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file $O/traffic_$R.csv python tools/profile_all.py \
    > $O/profile_order.log 2>&1
  log "ncu traffic rc=$?"
  python tools/ncu_summary.py traffic $O/traffic_$R.csv $O/profile_order.log $O/traffic.json
else
  log "profile_all failed: $(tail -3 $O/profile_order_plain.log)"
fi

log "launch list of the default bench command"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_$R.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 \
  > $O/launches_$R.log 2>&1
log "launch list rc=$?"

log "full captures: cfg4 (single-launch kernel) and cfg2 (panel kernel)"
if timeout 300 python tools/profile_one.py --config cfg4 --launches 2 > /dev/null 2>&1; then
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"lrb_varn" \
    -c 1 -f -o $O/ncu_cfg4_$R python tools/profile_one.py --config cfg4 --launches 2 \
    > $O/ncu_cfg4_$R.log 2>&1
  log "ncu cfg4 rc=$?"
fi
if timeout 300 python tools/profile_one.py --config cfg2 --launches 2 > /dev/null 2>&1; then
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"lrb_(gemm|panel)_kernel" \
    -c 1 -f -o $O/ncu_cfg2_$R python tools/profile_one.py --config cfg2 --launches 2 \
    > $O/ncu_cfg2_$R.log 2>&1
  log "ncu cfg2 rc=$?"
fi
if timeout 300 python tools/profile_all.py --only lr_r64_b2048 > /dev/null 2>&1; then
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"lrb_lowrank_big" \
    -c 1 -f -o $O/ncu_lr_r64_$R python tools/profile_all.py --only lr_r64_b2048 \
    > $O/ncu_lr_r64_$R.log 2>&1
  log "ncu lr_r64 rc=$?"
fi
if timeout 300 python tools/profile_all.py --only blr_n16384_b256_r16_k16 > /dev/null 2>&1; then
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"blr_fused" \
    -c 1 -f -o $O/ncu_blr_k16_$R python tools/profile_all.py --only blr_n16384_b256_r16_k16 \
    > $O/ncu_blr_k16_$R.log 2>&1
  log "ncu blr k16 rc=$?"
  # steady-state DRAM bytes of repeated launches (no cache flush between them)
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --cache-control none -k regex:"blr_fused" --csv \
    --log-file $O/blr_k16_warm_traffic_$R.csv python tools/profile_all.py \
    --only blr_n16384_b256_r16_k16 --repeat 6 > /dev/null 2>&1
  log "ncu blr warm traffic rc=$?"
fi
for f in ncu_cfg4_$R ncu_cfg2_$R ncu_lr_r64_$R ncu_blr_k16_$R; do
  [ -f $O/$f.ncu-rep ] && python tools/ncu_summary.py rep $O/$f.ncu-rep > $O/$f.json 2>> $O/probe_$R.err
done
log "smoke"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$R.txt 2>&1
log "smoke rc=$? $(tail -1 $O/smoke_$R.txt | cut -c1-200)"
log "done"
