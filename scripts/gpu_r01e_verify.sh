# re-entry check of HEAD: gpu tests, smoke, default bench line, reference arm
set -x
TAG=${TAG:-r01e}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -2 gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_${TAG}.err
ls gpurun_out
