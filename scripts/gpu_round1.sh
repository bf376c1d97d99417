set -x
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -5 gpurun_out/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e > gpurun_out/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 4 -c 1 -o gpurun_out/prof_main_n2048 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --seqlens 2048 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
