# round-2 evidence run: GPU tests, full bench line, ncu launch list + --set full captures (TAG)
TAG=${TAG:-r2_v1}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -4 > gpurun_out/${TAG}_pytest.txt
cat gpurun_out/${TAG}_pytest.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|combine|scatter|merge|quant" --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --legs "" > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_tc -c 2 -o gpurun_out/$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --legs "" > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/$TAG.ncu-rep
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"attn_tc|cm_merge" -s 4 -c 2 -o gpurun_out/${TAG}_layer python scripts/prof_layer.py > gpurun_out/${TAG}_layer.log 2>&1
ncu -i gpurun_out/${TAG}_layer.ncu-rep --page raw --csv > gpurun_out/${TAG}_layer_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_layer.ncu-rep
ls -la gpurun_out | grep $TAG
