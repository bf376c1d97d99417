# quick GPU iteration: parity subset + bench (sweep table) for the default workload
set -x
timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q -k "backward_matches or determinism_100 or sharding" 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -3 gpurun_out/bench_quick.err
