mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fp8.py -q -x --timeout 600 -k "cluster_merge or per_layer or kernel_options or graph" 2>&1 | tail -2
