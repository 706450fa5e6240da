#!/bin/bash
# One gpurun pass: GPU tests, smoke, bench line.
# Usage (on the box): bash scripts/gpu_check.sh [tag]
tag=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
tail -3 gpurun_out/gputests_$tag.log; cat gpurun_out/bench_$tag.json | head -c 600
