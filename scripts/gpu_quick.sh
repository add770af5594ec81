mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_parity.py -q -x --timeout 300 --timeout-method=thread -k "query or fp8 or needle or flash or sharded or negative" 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --legs fp8,split --no-cpu-baseline 2>/dev/null > gpurun_out/bench_quick.json
python -c "
import json; d=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1])
print('HEAD', d['query_latency_us_32_layers'], d['append_tflops'], d['kernel_ms'])
print('FP8', d['fp8_kv']['query_latency_us_32_layers'], d['fp8_kv']['append_tflops'], d['fp8_kv']['split_kv_128k'])
print('BF16_128k', d['split_kv_128k'])"
