set -x
DASH_VARIANT=7 timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -m gpu -x -q -k "64 or not 128" 2>&1 | tail -2
for v in 0 7 0 7; do
DASH_VARIANT=$v timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 64 causal
DASH_VARIANT=$v timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 64 full
done 2>&1 | grep DEBUG | tee gpurun_out/exp_r01e_v7.txt
