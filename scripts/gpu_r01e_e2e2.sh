set -x
for c in 4 8 16; do DASH_HOST_CHUNKS=$c timeout 600 python bench.py --no-sweep --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks', $c, d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
timeout 600 python -m pytest tests/test_gpu_bwd.py -m gpu -x -q -k "host" 2>&1 | tail -2
