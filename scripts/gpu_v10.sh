# v10: smem variant 1 (2 staging buffers) vs 0
set -x
DASH_VARIANT=2 timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -m gpu -x -q 2>&1 | tail -3
for var in 0 2; do
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 causal
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 full
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 64 causal
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 64 full
done 2>&1 | grep -E "DEBUG|VAR" | tee gpurun_out/exp_v10b.txt
