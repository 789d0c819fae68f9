run() { echo "flags=$1 $(LRB_DEBUG_FLAGS=$1 timeout 300 python bench.py --config $2 --no-cpu --e2e-steps 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['step_ms']['min'])")"; }
for f in 0 32 48 64 96 160 0; do run $f blr_n16384_b256_r16_k16; done
for f in 0 32 64; do run $f blr_n32768_b512_r8_k8; done
