# v8: deferred dQ issue order (default) vs legacy order (DASH_DEBUG=8)
set -x
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -m gpu -x -q 2>&1 | tail -3
for dbg in 0 8; do
  DASH_DEBUG=$dbg timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 causal
  DASH_DEBUG=$dbg timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 full
  DASH_DEBUG=$dbg timeout 300 python scripts/exp_reduce_path.py 2048,16384 64 causal
done 2>&1 | grep DEBUG | tee gpurun_out/exp_v8.txt
