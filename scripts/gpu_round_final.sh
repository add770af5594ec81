# Round-end evidence: smoke, GPU tests, bench line, ncu launch list and one --set full capture
# of the bench step's two attention launches (append, query).  TAG names the profile set.
set -x
TAG=${TAG:-r1_v5}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread 2>&1 | tail -8
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 2000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|combine|scatter|merge|quant" --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --legs "" > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_tc -c 2 -o gpurun_out/$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --legs "" > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/$TAG.ncu-rep
ls -la gpurun_out
