# ncu --set full with source of the main kernel (N=2048 causal, auto) + full pipeline traces
set -x
TAG=${TAG:-r01e}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 2 -c 1 -o gpurun_out/prof_${TAG}_n2048 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --seqlens 2048 > gpurun_out/ncu_full_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}_n2048.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_n2048.csv 2>&1
ncu -i gpurun_out/prof_${TAG}_n2048.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_n2048.csv 2>&1
for s in shift descending; do timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule $s --out gpurun_out/trace_${TAG}_$s.json --npz gpurun_out/trace_${TAG}_$s.npz > /dev/null; done
timeout 120 python scripts/trace_pipeline.py --seqlen 16384 --schedule descending --out gpurun_out/trace_${TAG}_16k_desc.json --npz gpurun_out/trace_${TAG}_16k_desc.npz > /dev/null
DASH_DEBUG=5 timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_${TAG}_shift_dbg5.json --npz gpurun_out/trace_${TAG}_shift_dbg5.npz > /dev/null
ls -la gpurun_out
