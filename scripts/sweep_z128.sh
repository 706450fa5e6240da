#!/bin/bash
# K3 at Pz = 128 (block 2048x2048x64, 64^3 cubes): register budget sweep (run under gpurun).
cp paper_1411_2565_b200/libgrace.so /tmp/libgrace_base.so
for v in "$@"; do
  GRACE_NVCC_FLAGS="$v" python paper_1411_2565_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"
  python bench.py --workload block_2048x2048x64 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('block', '%.3f ms/step' % d['ms_per_step'], ' '.join('%s=%.3f' % (k, v['ms_per_launch']) for k, v in d['kernels'].items()))"
  timeout 300 python scripts/small_cube_kernels.py 64 2>&1
done
cp /tmp/libgrace_base.so paper_1411_2565_b200/libgrace.so
