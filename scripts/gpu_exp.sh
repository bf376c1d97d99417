set -x
for dbg in 0 1; do DASH_DEBUG=$dbg timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_dbg$dbg.json 2>/dev/null; DASH_DEBUG=$dbg timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule naive --atomic --out gpurun_out/trace_dbg$dbg.json > /dev/null; done
