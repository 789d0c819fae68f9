#!/usr/bin/env bash
# Both arms of every widened-row bench config (low-rank product, BLR matvec)
# into gpurun_out/bench_rows_$1.jsonl (GPU arm then reference arm per config).
R=${1:-r02}
O=gpurun_out
mkdir -p $O
: > $O/bench_rows_$R.jsonl
for c in lr_r8_b1024 lr_r15_b1024 lr_r16_b1024 lr_r32_b2048 lr_r64_b2048 lr_r96_b1024 lr_r128_b1024 \
         blr_n32768_b512_r8_k8 blr_n16384_b256_r16_k16 blr_n16384_b512_r32_k16 blr_n32768_b512_r8_k1 \
         lrx_m512_r8 lrx_m512_r32 blrd_n16384_b512_r16; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 2>> $O/bench_rows_$R.err | tail -1 >> $O/bench_rows_$R.jsonl
  timeout 900 python bench.py --config $c --impl reference --steps 3 --warmup 3 2>> $O/bench_rows_$R.err | tail -1 >> $O/bench_rows_$R.jsonl
done
echo "rows: $(wc -l < $O/bench_rows_$R.jsonl)"
