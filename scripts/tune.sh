#!/bin/bash
# Rebuild libgrace with each tile variant and print per-kernel times (run on a GPU box).
# usage: scripts/tune.sh "-DGRACE_Y_ELEMS=8192" "-DGRACE_Y_ELEMS=16384 -DGRACE_EPT=8" ...
for v in "$@"; do
  GRACE_NVCC_FLAGS="$v" python paper_1411_2565_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '%.3f ms/step' % d['ms_per_step'], ' '.join('%s=%.3f' % (k, v['ms_per_launch']) for k, v in d['kernels'].items()))"
done
