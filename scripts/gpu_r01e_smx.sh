# softmax: diagonal-only masking
set -x
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 64 causal
timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 64 full
timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 causal
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --head-dim 64 --schedule shift --out gpurun_out/trace_r01e_d64b_shift.json --npz gpurun_out/trace_r01e_d64b_shift.npz > /dev/null
