# One ncu --set full capture of the first attn_tc launch (data-plane append) with
# SASS-level source export (stall sampling per instruction) + raw page.
set -x
mkdir -p gpurun_out
TAG=${TAG:-prof}
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_tc -c ${COUNT:-1} -o gpurun_out/$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --legs "" > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ls -la gpurun_out
