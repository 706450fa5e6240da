#!/bin/bash
# K3 occupancy / tile sweep (run under gpurun); restores the base build afterwards.
cp paper_1411_2565_b200/libgrace.so /tmp/libgrace_base.so
GRACE_PTXAS_V=1 GRACE_NVCC_FLAGS="-DGRACE_MINB_Z=5" python paper_1411_2565_b200/build.py --force 2>&1 | grep -A2 "k3_z" | grep -i "registers\|spill" > gpurun_out/sweep_k3_ptxas.txt
bash scripts/tune.sh "" "-DGRACE_MINB_Z=5" "-DGRACE_MINB_Z=6" "-DGRACE_Z_MINNT=256 -DGRACE_ZB=32 -DGRACE_MINB_Z=2" > gpurun_out/sweep_k3.txt 2>&1
cp /tmp/libgrace_base.so paper_1411_2565_b200/libgrace.so
