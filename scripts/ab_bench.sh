# A/B helper: the headline step three times (append TFLOP/s, query latency), plus the fp8 leg once
mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --legs "" --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('AB', round(d['append_tflops'],1), round(d['query_latency_us_32_layers'],1), {k: round(v,4) for k,v in d['kernel_ms'].items()})"; done
