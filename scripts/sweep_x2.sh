#!/bin/bash
# x-kernel tile / CTAs-per-SM sweep over the workloads (run under gpurun); restores the base build afterwards.
cp paper_1411_2565_b200/libgrace.so /tmp/libgrace_base.so
for v in "$@"; do
  GRACE_NVCC_FLAGS="$v" python paper_1411_2565_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for w in slab_1024x1024x32 film_512x512x8 sp4_field1 block_2048x2048x64; do
    st=40; [ $w = block_2048x2048x64 ] && st=10; [ $w = sp4_field1 ] && st=2000
    python bench.py --workload $w --steps $st --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$w', '%.4f ms/step' % d['ms_per_step'], ' '.join('%s=%.4f' % (k, v['ms_per_launch']) for k, v in d['kernels'].items()))"
  done
done
cp /tmp/libgrace_base.so paper_1411_2565_b200/libgrace.so
