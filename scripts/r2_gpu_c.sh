timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -q -x --timeout 300 -k "llama or query_lengths or needle or flash or batch or negative or cluster or fp8_create or per_layer" 2>&1 | tail -2
bash scripts/ab_variants.sh prev
