#!/bin/bash
# Bench the default build under different environment settings, interleaved.
# Usage (on the box): bash scripts/sweep_env.sh OUT "VAR=a VAR=b ..." [workload] [reps]
out=$1; vs=$2; wl=${3:-slab_1024x1024x32}; reps=${4:-2}
mkdir -p gpurun_out; : > gpurun_out/$out
for r in $(seq $reps); do
  for v in $vs; do
    env $v timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), {k: round(v['ms_per_launch'],4) for k, v in d['kernels'].items()})" >> gpurun_out/$out
  done
done
cat gpurun_out/$out
