set -x
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 5000 gpurun_out/bench.json; tail -20 gpurun_out/bench.err
