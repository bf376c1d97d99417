# v13: full GPU tests + bench for all four sweep configurations (W automatic)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v13_causal128.json 2> gpurun_out/bench_v13.err; tail -2 gpurun_out/bench_v13.err
timeout 900 python bench.py --steps 10 --warmup 3 --full --no-cpu --no-e2e > gpurun_out/bench_v13_full128.json 2>> gpurun_out/bench_v13.err
timeout 900 python bench.py --steps 10 --warmup 3 --head-dim 64 --no-cpu --no-e2e > gpurun_out/bench_v13_causal64.json 2>> gpurun_out/bench_v13.err
timeout 900 python bench.py --steps 10 --warmup 3 --head-dim 64 --full --no-cpu --no-e2e > gpurun_out/bench_v13_full64.json 2>> gpurun_out/bench_v13.err
tail -3 gpurun_out/bench_v13.err
