LAYER_APPEND=0 LAYER_CFGS="0,1,4 0,1,2 0,1,4 0,1,2 0,1,4 0,1,2 0,1,4 0,1,2 0,1,4 0,1,2 0,1,4 0,1,2" timeout 900 python scripts/layer_probe.py 2>&1 | grep "graph" | awk '{print $2, $5, $7}'
