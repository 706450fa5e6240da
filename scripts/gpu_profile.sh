#!/bin/bash
# ncu evidence for profiles/: the launch list (gpu__time_duration of every
# launch, cold and serialised) and one --set full capture of the six step kernels.
# Usage (on the box): bash scripts/gpu_profile.sh TAG [workload]
tag=${1:-x}
wl=${2:-slab_1024x1024x32}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1_$tag.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_x_bulk|k_y_stage|k_y_tma|k3_z|k6_llg|k2f_y|k5_inv' -c 6 -f -o gpurun_out/prof_$tag \
  python bench.py --workload $wl --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2_$tag.log 2>&1
echo "profile rc=$?"
