# early claim of the next job (producer prefetch) vs claim after the last release
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for pf in 0 1 0 1; do
  DASH_NO_PREFETCH=$pf timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 128 causal
  DASH_NO_PREFETCH=$pf timeout 300 python scripts/exp_reduce_path.py 512,2048,8192,16384 128 full
  DASH_NO_PREFETCH=$pf timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 64 causal
  DASH_NO_PREFETCH=$pf timeout 300 python scripts/exp_reduce_path.py 2048,4096,8192 64 full
done 2>&1 | grep -E "DEBUG|PF" | tee gpurun_out/exp_r01e_pf.txt
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_r01e_pf_shift.json --npz gpurun_out/trace_r01e_pf_shift.npz > /dev/null
