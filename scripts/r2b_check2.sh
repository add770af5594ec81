mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fp8.py -q -x --timeout 600 -k "cluster_merge or per_layer or kernel_options or batch or flash" 2>&1 | tail -3
VARS="base" LAYER_APPEND=0 bash scripts/r2b_early.sh 2>&1 | tail -2
timeout 600 python bench.py --legs nsweep --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps(d['context_sweep'])[:2500])"
