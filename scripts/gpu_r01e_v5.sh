# V=5 (3-slot half-unit staging ring + single dS^T buffer) vs V=3; traces with the new stamps
set -x
DASH_VARIANT=5 timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -3
for var in 3 5 3 5; do
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,4096,16384 128 causal
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,4096,16384 128 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_r01e_v5.txt
for var in 3 5; do DASH_VARIANT=$var timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_r01e_v${var}b_shift.json --npz gpurun_out/trace_r01e_v${var}b_shift.npz > /dev/null; done
