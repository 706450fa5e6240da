#!/bin/bash
# Bench line, ncu launch list and one ncu --set full capture of the step kernels (run under gpurun).
set -e
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_x_bulk|k1_fwd|k_y_tma|k_y_stage|k3_z|k5_inv|k6_llg" -c 6 -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
