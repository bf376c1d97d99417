timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule naive --atomic --out gpurun_out/trace_atomic.json > /dev/null
timeout 120 python scripts/trace_pipeline.py --seqlen 16384 --schedule shift --out gpurun_out/trace_shift16k.json > /dev/null
