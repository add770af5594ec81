mkdir -p gpurun_out
python scripts/qkv_once.py 256 32 && echo plain-ok
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qkv_rope -c 2 -o gpurun_out/qkv_r2b -f python scripts/qkv_once.py 256 32 > gpurun_out/qkv_ncu.log 2>&1; echo ncu exit $?
tail -3 gpurun_out/qkv_ncu.log
