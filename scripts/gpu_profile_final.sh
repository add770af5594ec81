# Launch list of the bench step and one --set full capture of its two attention launches (TAG).
TAG=${TAG:-r1_v6}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|combine|scatter|merge|quant" --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --legs "" > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_tc -c 2 -o gpurun_out/$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --legs "" > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/$TAG.ncu-rep
ls -la gpurun_out | grep $TAG
