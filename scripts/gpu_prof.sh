set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|combine|scatter" --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_tc -c 2 -o gpurun_out/prof_tc_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_tc_r1.log 2>&1
ls -la gpurun_out
