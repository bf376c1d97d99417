# pipelined host path: bit test + e2e bench
set -x
timeout 600 python -m pytest tests/test_gpu_bwd.py -m gpu -x -q -k "host or determinism" 2>&1 | tail -3
timeout 600 python bench.py --no-sweep --no-cpu > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; tail -2 gpurun_out/bench_e2e.err
python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value'], d['e2e'])"
