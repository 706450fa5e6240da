#!/bin/bash
# Small-row x-kernel configuration sweep on the Table-1 cubes (run under gpurun); restores the base build.
cp paper_1411_2565_b200/libgrace.so /tmp/libgrace_base.so
for v in "$@"; do
  GRACE_NVCC_FLAGS="$v" python paper_1411_2565_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"; python scripts/small_cube_kernels.py 8 16 32 2>&1
done
cp /tmp/libgrace_base.so paper_1411_2565_b200/libgrace.so
