mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qkv.py -q -x --timeout 300 2>&1 | tail -3
timeout 300 python scripts/qkv_trace.py 2>&1 | tail -24
timeout 600 python bench.py --legs qkv --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps(d['qkv_rope']))"
