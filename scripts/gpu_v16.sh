# v16: variant 3 with half-pipelined staging (default) vs variant 0
set -x
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -m gpu -x -q 2>&1 | tail -3
for var in 3 0; do
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 causal
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_v17.txt
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_v17_shift.json > /dev/null
