# abort-flag polling every 16 misses (was: every miss) -- correctness + timing + trace
set -x
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do
  timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 128 causal
  timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 128 full
  timeout 300 python scripts/exp_reduce_path.py 2048,16384 64 causal
  timeout 300 python scripts/exp_reduce_path.py 2048,4096,8192 64 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_r01e_abort.txt
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_r01e_ab_shift.json --npz gpurun_out/trace_r01e_ab_shift.npz > /dev/null
