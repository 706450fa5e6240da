#!/bin/bash
# Rebuild with each flag variant and print scripts/kernel_split.py for the given workloads.
# usage: WL="cube:128 film_512x512x8" scripts/tune_split.sh "" "-DFOO=1" ...
for v in "$@"; do
  GRACE_NVCC_FLAGS="$v" python paper_1411_2565_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"
  python scripts/kernel_split.py ${WL:-slab_1024x1024x32}
done
