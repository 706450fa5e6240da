#!/bin/bash
# K3 for long z pencils (Pz = 256..1024: 128^3..512^3 cubes): tile / register budget sweep (run under gpurun).
cp paper_1411_2565_b200/libgrace.so /tmp/libgrace_base.so
for v in "$@"; do
  GRACE_NVCC_FLAGS="$v" python paper_1411_2565_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"; timeout 300 python scripts/small_cube_kernels.py 128 256 512 2>&1
done
cp /tmp/libgrace_base.so paper_1411_2565_b200/libgrace.so
