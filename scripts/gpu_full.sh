# full GPU check: all gpu tests, smoke, pipeline traces, bench, ncu launch list
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python __graft_entry__.py smoke 2>&1 | tail -1
for s in shift naive; do timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule $s --out gpurun_out/trace_$s.json > /dev/null; done
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule naive --atomic --out gpurun_out/trace_atomic.json > /dev/null
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e > /dev/null 2>&1
