mkdir -p gpurun_out
timeout 600 ncu --section WarpStateStats --section SourceCounters --warp-sampling-interval 0 --import-source on --clock-control none -k regex:qkv_rope -c 1 -o gpurun_out/qkv_r2b2 -f python scripts/qkv_once.py 256 > gpurun_out/qkv_ncu2.log 2>&1; echo ncu exit $?
ncu -i gpurun_out/qkv_r2b2.ncu-rep --page source --csv --print-source sass > gpurun_out/qkv_r2b2_sass.csv 2>/dev/null
rm -f gpurun_out/qkv_r2b2.ncu-rep
