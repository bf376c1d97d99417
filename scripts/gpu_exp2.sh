set -x
for dbg in 0 2; do DASH_DEBUG=$dbg timeout 300 python bench.py --steps 5 --warmup 2 --full --no-cpu --no-e2e > gpurun_out/bench_full_dbg$dbg.json 2>/dev/null; done
DASH_DEBUG=2 timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_causal_dbg2.json 2>/dev/null
for s in naive shift; do timeout 120 python scripts/trace_pipeline.py --seqlen 4096 --full --schedule $s --out gpurun_out/trace_full_$s.json > /dev/null; done
