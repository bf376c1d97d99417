set -x
timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -2
for dbg in 0 4; do DASH_DEBUG=$dbg timeout 300 python bench.py --steps 5 --warmup 2 --full --no-cpu --no-e2e > gpurun_out/bench_full_dbg$dbg.json 2>/dev/null; DASH_DEBUG=$dbg timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_causal_dbg$dbg.json 2>/dev/null; done
timeout 120 python scripts/trace_pipeline.py --seqlen 4096 --full --schedule shift --out gpurun_out/trace_full_shift.json > /dev/null
