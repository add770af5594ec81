# Launch-phase timeline of the per-layer query (build first: scripts/build_gtrace.sh);
# GT_CFGS = "cluster,merge ..." settings (SSA_OPT_CLUSTER, SSA_OPT_CM_MERGE)
cp variants/gtrace/libssa.so paper_2605_13784_b200/libssa.so
GT_CFGS="${GT_CFGS:-0,2}" timeout 600 python scripts/gtrace_run.py 2>&1 | grep GT
