# round-2 evidence: full GPU suite, smoke, bench line, ncu launch list + full captures (TAG)
TAG=${TAG:-r2_v2}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -q -m gpu --timeout 900 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|combine|scatter|merge|quant" --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --legs "" > /dev/null 2>&1; echo "launches exit $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_tc -c 2 -o gpurun_out/$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --legs "" > gpurun_out/$TAG.log 2>&1; echo "full exit $?"
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/$TAG.ncu-rep
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc -s 3 -c 1 -o gpurun_out/${TAG}_layer python scripts/prof_layer.py > gpurun_out/${TAG}_layer.log 2>&1; echo "layer exit $?"
ncu -i gpurun_out/${TAG}_layer.ncu-rep --page raw --csv > gpurun_out/${TAG}_layer_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_layer.ncu-rep
ls -la gpurun_out | grep $TAG
