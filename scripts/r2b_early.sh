# per-layer query under early-stage variants (interleaved: base, e1, e2, base)
cp paper_2605_13784_b200/libssa.so /tmp/base_libssa.so
for v in ${VARS:-base early1 early2 base early1 early2}; do
  if [ $v = base ]; then cp /tmp/base_libssa.so paper_2605_13784_b200/libssa.so; else cp variants/$v/libssa.so paper_2605_13784_b200/libssa.so; fi
  LAYER_APPEND=0 LAYER_CFGS="0,1,2" timeout 300 python scripts/layer_probe.py 2>&1 | grep -E "graph" | grep -v append | sed "s/^/$v /"
done
