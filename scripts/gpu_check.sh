#!/bin/bash
# One gpurun pass: GPU tests, smoke, bench line, memcheck of the small cases.
# Usage (on the box): bash scripts/gpu_check.sh [tag]
tag=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 900 compute-sanitizer --tool memcheck --leak-check no python scripts/memcheck_small.py > gpurun_out/memcheck_$tag.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_$tag.log
tail -3 gpurun_out/gputests_$tag.log; cat gpurun_out/bench_$tag.json | head -c 600; tail -3 gpurun_out/memcheck_$tag.log
