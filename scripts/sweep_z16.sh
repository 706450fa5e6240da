#!/bin/bash
# K3 / K2' at L = 16 (film Pz, 8^3 cubes): CTAs-per-SM register budget sweep (run under gpurun); restores the base build.
cp paper_1411_2565_b200/libgrace.so /tmp/libgrace_base.so
for v in "$@"; do
  GRACE_NVCC_FLAGS="$v" python paper_1411_2565_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"
  python bench.py --workload film_512x512x8 --steps 200 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('film', '%.4f ms/step' % d['ms_per_step'], ' '.join('%s=%.4f' % (k, v['ms_per_launch']) for k, v in d['kernels'].items()))"
  python scripts/small_cube_kernels.py 8 2>&1
done
cp /tmp/libgrace_base.so paper_1411_2565_b200/libgrace.so
