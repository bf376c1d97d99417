# BASELINE configs 3-5 (full-mask sweeps, long context, model check)
set -x
timeout 600 python bench.py --steps 5 --warmup 2 --full --no-cpu --no-e2e > gpurun_out/bench_full_hd128.json 2>gpurun_out/bench_full_hd128.err
timeout 600 python bench.py --steps 5 --warmup 2 --full --head-dim 64 --no-cpu --no-e2e > gpurun_out/bench_full_hd64.json 2>gpurun_out/bench_full_hd64.err
timeout 600 python bench.py --steps 5 --warmup 2 --head-dim 64 --no-cpu --no-e2e > gpurun_out/bench_causal_hd64.json 2>gpurun_out/bench_causal_hd64.err
timeout 900 python scripts/long_context.py --out gpurun_out/long_context.json > gpurun_out/long_context.log 2>&1
timeout 900 python scripts/model_check.py --out gpurun_out/model_check.json > gpurun_out/model_check.log 2>&1
tail -3 gpurun_out/*.err gpurun_out/long_context.log gpurun_out/model_check.log
