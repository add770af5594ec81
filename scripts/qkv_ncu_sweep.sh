# ncu per-launch duration of the fused projection: debug modes x split factors
# (1 mainloop+dump, 4 no MMA, 5 no TMA loads)
mkdir -p gpurun_out
for cfg in "1 2 256" "4 2 256" "5 2 256" "1 5 32" "4 5 32" "5 5 32" "0 2 256" "0 5 32"; do
  set -- $cfg
  SSA_QKV_DEBUG=$1 SSA_QKV_SPLITS=$2 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg --clock-control none -k regex:qkv --csv python scripts/qkv_probe.py $3 2>/dev/null | grep qkv | awk -F'","' -v c="$cfg" '{print "dbg S m = "c": "$(NF-2)" "$(NF)}'
done
