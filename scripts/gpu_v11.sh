# v11: interleaved accumulators W=2 vs W=1
set -x
DASH_ACC_SPLIT=2 timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -m gpu -x -q 2>&1 | tail -3
for w in 1 2; do
  DASH_ACC_SPLIT=$w timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 causal
  DASH_ACC_SPLIT=$w timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 full
  DASH_ACC_SPLIT=$w timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 64 causal
  DASH_ACC_SPLIT=$w timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 64 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_v11.txt
