#!/bin/bash
# Round-end evidence on one box: GPU tests + smoke + bench, ncu launch list and
# full capture, film bench, cuFFT comparison, Table-1 sweep, KP sweep.
# Usage (on the box): bash scripts/final_evidence.sh TAG
bash scripts/gpu_check.sh ${1:-f4}
bash scripts/gpu_profile.sh ${1:-f4}
timeout 300 python bench.py --workload film_512x512x8 --steps 50 --warmup 5 > gpurun_out/bench_film_${1:-f4}.json 2>/dev/null
(timeout 300 python bench_cufft.py --workload slab_1024x1024x32; timeout 300 python bench_cufft.py --workload film_512x512x8) > gpurun_out/cufft_${1:-f4}.json 2>/dev/null
timeout 1500 python scripts/table1_sweep.py --out gpurun_out/t1_${1:-f4} > gpurun_out/t1_${1:-f4}.log 2>&1
timeout 600 python scripts/plane_sweep.py --out gpurun_out/plane_sweep_${1:-f4}.json > /dev/null 2>&1
echo done
