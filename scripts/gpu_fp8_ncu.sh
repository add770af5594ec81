mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -c 1 -o gpurun_out/fp8_query -f python scripts/fp8_probe.py > gpurun_out/fp8_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -c 1 -o gpurun_out/bf16_query -f python scripts/fp8_probe.py bf16 >> gpurun_out/fp8_ncu.log 2>&1
tail -3 gpurun_out/fp8_ncu.log
