# Per-layer query under early-pool-stage variants, interleaved (VARS; default base, early1,
# early2 twice).  Build the variants first: scripts/build_variant.sh earlyN -DSSA_EARLY_STAGES=N
cp paper_2605_13784_b200/libssa.so /tmp/base_libssa.so
for v in ${VARS:-base early1 early2 base early1 early2}; do
  if [ $v = base ]; then cp /tmp/base_libssa.so paper_2605_13784_b200/libssa.so; else cp variants/$v/libssa.so paper_2605_13784_b200/libssa.so; fi
  LAYER_APPEND=0 LAYER_CFGS="0,1,2" timeout 300 python scripts/layer_probe.py 2>&1 | grep -E "graph" | grep -v append | sed "s/^/$v /"
done
