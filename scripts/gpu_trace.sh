set -x
timeout 300 python -m pytest tests/test_gpu_bwd.py -x -q -k "backward_matches or determinism_100" 2>&1 | tail -3
for s in shift naive; do timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule $s --out gpurun_out/trace_$s.json > /dev/null 2>gpurun_out/trace_$s.err; done
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule naive --atomic --out gpurun_out/trace_atomic.json > /dev/null 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -3 gpurun_out/bench_quick.err
