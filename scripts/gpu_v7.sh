# v7 check: fused finalise + replay tests, reduction-path timing experiments
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
for dbg in 0 1 5; do  # 5 = no staging, no reduce
  DASH_DEBUG=$dbg timeout 300 python scripts/exp_reduce_path.py 2048,16384 128 causal
  DASH_DEBUG=$dbg timeout 300 python scripts/exp_reduce_path.py 2048,16384 128 full
done 2>&1 | grep DEBUG | tee gpurun_out/exp_v7b.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v7b.json 2> gpurun_out/bench_v7b.err; tail -3 gpurun_out/bench_v7b.err
