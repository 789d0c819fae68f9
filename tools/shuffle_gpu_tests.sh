#!/usr/bin/env bash
# Run the GPU test files in several orders (reverse, then seeded shuffles) in
# ONE process each, to catch failures that depend on what ran before (stale
# pool memory, neighbouring allocations, leftover context state).
#   gpurun -- 'bash tools/shuffle_gpu_tests.sh 3'
N=${1:-3}
files=$(ls tests/test_gpu_*.py)
echo "== reverse"
timeout 900 python -m pytest $(echo $files | tr ' ' '\n' | sort -r | tr '\n' ' ') -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for seed in $(seq 1 $N); do
  echo "== shuffle seed $seed"
  order=$(python - "$seed" $files <<'PY'
import random, sys
seed, files = int(sys.argv[1]), sys.argv[2:]
random.Random(seed).shuffle(files)
print(" ".join(files))
PY
)
  echo "$order"
  timeout 900 python -m pytest $order -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
done
