# final round-1 measurements: tests, smoke, the four sweep configurations, launch list, DRAM traffic, configs 4-5
set -x
TAG=${TAG:-r01i}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -2 gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --full --no-cpu --no-e2e > gpurun_out/bench_${TAG}_full128.json 2>> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --head-dim 64 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_causal64.json 2>> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --head-dim 64 --full --no-cpu --no-e2e > gpurun_out/bench_${TAG}_full64.json 2>> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dash_bwd_kernel -c 6 --csv --log-file gpurun_out/dram_${TAG}.csv python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 2 -c 1 -o gpurun_out/prof_${TAG}_n2048 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --seqlens 2048 > gpurun_out/ncu_full_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}_n2048.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_n2048.csv 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 900 python scripts/long_context.py --out gpurun_out/long_context_${TAG}.json > gpurun_out/long_context_${TAG}.log 2>&1; tail -2 gpurun_out/long_context_${TAG}.log
timeout 1200 python scripts/model_check.py --out gpurun_out/model_check_${TAG}.json > gpurun_out/model_check_${TAG}.log 2>&1; tail -2 gpurun_out/model_check_${TAG}.log
ls gpurun_out | grep ${TAG}
