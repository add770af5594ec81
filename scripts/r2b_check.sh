mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 600 -k "cluster_merge or per_layer" 2>&1 | tail -3
LAYER_CFGS="0,1,2" timeout 600 python scripts/layer_probe.py 2>&1 | grep LAYER
