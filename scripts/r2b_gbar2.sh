mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "cluster_merge" 2>&1 | tail -3
LAYER_CFGS="0,1,1 0,1,2" timeout 600 python scripts/layer_probe.py 2>&1 | grep LAYER
cp variants/gtrace/libssa.so paper_2605_13784_b200/libssa.so
GT_CFGS="0,2" timeout 600 python scripts/gtrace_run.py 2>&1 | grep GT
