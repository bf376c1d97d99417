# V=6 (split reduction: half bulk engine, half red.global from the drain) vs V=3
set -x
DASH_VARIANT=6 timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -3
for var in 3 6 3 6; do
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,4096,16384 128 causal
  DASH_VARIANT=$var timeout 300 python scripts/exp_reduce_path.py 512,2048,4096,16384 128 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_r01e_v6.txt
DASH_VARIANT=6 timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_r01e_v6_shift.json --npz gpurun_out/trace_r01e_v6_shift.npz > /dev/null
