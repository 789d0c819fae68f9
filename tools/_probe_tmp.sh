run() { echo "flags=$1 $(LRB_DEBUG_FLAGS=$1 timeout 300 python bench.py --config $2 --no-cpu --e2e-steps 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['step_ms']['min'])")"; }
timeout 900 python -m pytest tests/test_gpu_blr.py -x -q -m gpu 2>&1 | tail -3
for f in 0 128 1024 2080 16; do run $f blr_n16384_b256_r16_k16; done
for f in 0 128; do run $f blr_n32768_b512_r8_k8; done
