set -x
timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -2
for s in shift; do timeout 120 python scripts/trace_pipeline.py --seqlen 4096 --full --schedule $s --out gpurun_out/trace_full_$s.json > /dev/null; done
timeout 120 python scripts/trace_pipeline.py --seqlen 4096 --full --schedule naive --atomic --out gpurun_out/trace_full_atomic.json > /dev/null
timeout 300 python bench.py --steps 5 --warmup 2 --full --no-cpu --no-e2e > gpurun_out/bench_full_dbg0.json 2>/dev/null
timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_causal_dbg0.json 2>/dev/null
