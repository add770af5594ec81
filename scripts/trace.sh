# Per-tile SSA_TRACE timeline of the bench append + query, bf16 and E4M3 stores
# (build first: scripts/build_variant.sh trace -DSSA_TRACE; read with scripts/trace_stats.py)
cp variants/trace/libssa.so paper_2605_13784_b200/libssa.so
for kv in bf16 e4m3; do KV=$kv timeout 300 python scripts/trace_run.py 2>&1 | tail -2; done
ls gpurun_out/trace*
