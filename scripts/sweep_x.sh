#!/bin/bash
# K1/K5 x-kernel tile / occupancy sweep (run under gpurun); restores the base build afterwards.
cp paper_1411_2565_b200/libgrace.so /tmp/libgrace_base.so
bash scripts/tune.sh "" "-DGRACE_XB_ELEMS=4096 -DGRACE_XB_MINB=2" "-DGRACE_XB_ELEMS=2048 -DGRACE_XB_MINB=4" "-DGRACE_XB_ELEMS=4096 -DGRACE_XB_MINB=1" > gpurun_out/sweep_x.txt 2>&1
cp /tmp/libgrace_base.so paper_1411_2565_b200/libgrace.so
