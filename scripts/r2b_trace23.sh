cp variants/traceq23/libssa.so paper_2605_13784_b200/libssa.so
KV=bf16 timeout 300 python scripts/trace_run.py 2>&1 | tail -1
for k in append query; do mv gpurun_out/trace_bf16_$k.npy gpurun_out/trace23_bf16_$k.npy; done
