# v15: variant 3 (linear staging, 1-D bulk reduce) vs 0
set -x
DASH_VARIANT=3 timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -m gpu -x -q 2>&1 | tail -3
for var in 0 3; do
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 causal
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_v15.txt
DASH_VARIANT=3 timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_v15_shift.json > /dev/null
