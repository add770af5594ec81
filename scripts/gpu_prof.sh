set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|combine|scatter|merge" --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --legs "" > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:attn_tc -c 2 -o gpurun_out/prof_tc_r1b python bench.py --steps 1 --warmup 3 --no-cpu-baseline --legs "" > gpurun_out/prof_tc_r1b.log 2>&1
ls -la gpurun_out
