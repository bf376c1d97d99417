# full check: gpu tests, smoke, the four sweep configurations, launch list
set -x
TAG=${TAG:-r01e}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -2 gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --full --no-cpu --no-e2e > gpurun_out/bench_${TAG}_full128.json 2>> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --head-dim 64 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_causal64.json 2>> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --head-dim 64 --full --no-cpu --no-e2e > gpurun_out/bench_${TAG}_full64.json 2>> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e > /dev/null 2>&1
for s in shift descending; do timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule $s --out gpurun_out/trace_${TAG}_$s.json --npz gpurun_out/trace_${TAG}_$s.npz > /dev/null; done
ls gpurun_out
