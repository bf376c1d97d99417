timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule naive --atomic --out gpurun_out/trace_atomic.json > /dev/null
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --out gpurun_out/trace_shift.json > /dev/null
