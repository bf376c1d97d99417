# v8 evidence: ncu --set full (N=2048 shift, N=16384 descending), DRAM traffic per launch, configs 4 and 5
set -x
TAG=${TAG:-r01h}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 2 -c 1 -o gpurun_out/prof_${TAG}_n2048 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --seqlens 2048 > gpurun_out/ncu_full_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 2 -c 1 -o gpurun_out/prof_${TAG}_n16384 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --seqlens 16384 > gpurun_out/ncu_full16k_${TAG}.log 2>&1
for f in n2048 n16384; do ncu -i gpurun_out/prof_${TAG}_$f.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_$f.csv 2>&1; done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dash_bwd_kernel -c 6 --csv --log-file gpurun_out/dram_${TAG}.csv python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 python scripts/long_context.py --out gpurun_out/long_context_${TAG}.json > gpurun_out/long_context_${TAG}.log 2>&1; tail -3 gpurun_out/long_context_${TAG}.log
timeout 1200 python scripts/model_check.py --out gpurun_out/model_check_${TAG}.json > gpurun_out/model_check_${TAG}.log 2>&1; tail -3 gpurun_out/model_check_${TAG}.log
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
