# head grouping G: correctness under forced G, timing for G in 1,2,4,8 at short sequences
set -x
DASH_HEAD_GROUP=2 timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -3
DASH_HEAD_GROUP=4 timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -3
for g in 1 2 4 8; do
  DASH_HEAD_GROUP=$g timeout 300 python scripts/exp_reduce_path.py 512,1024,2048,4096 128 causal
  DASH_HEAD_GROUP=$g timeout 300 python scripts/exp_reduce_path.py 512,1024,2048,4096 128 full
  DASH_HEAD_GROUP=$g timeout 300 python scripts/exp_reduce_path.py 512,2048,4096 64 causal
  DASH_HEAD_GROUP=$g timeout 300 python scripts/exp_reduce_path.py 512,2048,4096 64 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_r01e_hg.txt
