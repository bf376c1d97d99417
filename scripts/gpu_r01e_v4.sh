# V=4 (4-part linear staging ring) vs V=3 (2 halves): correctness, timing, trace
set -x
DASH_VARIANT=4 timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_bwd.py -m gpu -x -q -k "128 or not d" 2>&1 | tail -3
for var in 3 4 3 4; do
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 128 causal
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 128 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_r01e_v4.txt
DASH_VARIANT=4 timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_r01e_v4_shift.json --npz gpurun_out/trace_r01e_v4_shift.npz > /dev/null
