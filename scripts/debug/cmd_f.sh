for i in 1 2 3; do python -m pytest tests/test_gpu_dist.py -q -x -k "nccl_path_one_rank_matches_single" 2>&1 | tail -1; done > gpurun_out/dbg_f.log
for i in 1 2 3; do GRACE_NO_PDL=1 python -m pytest tests/test_gpu_dist.py -q -x -k "nccl_path_one_rank_matches_single" 2>&1 | tail -1; done >> gpurun_out/dbg_f.log
for i in 1 2 3; do GRACE_NO_PIPE=1 python -m pytest tests/test_gpu_dist.py -q -x -k "nccl_path_one_rank_matches_single" 2>&1 | tail -1; done >> gpurun_out/dbg_f.log
python -m pytest tests/test_gpu_dist.py -q 2>&1 | tail -3 >> gpurun_out/dbg_f.log
GRACE_NO_PDL=1 python -m pytest tests/test_gpu_dist.py -q 2>&1 | tail -3 >> gpurun_out/dbg_f.log
