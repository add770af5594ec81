set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp8.py -q -x --timeout 240 --timeout-method=thread 2>&1 | tail -25
timeout 600 python bench.py --steps 5 --warmup 3 --legs fp8 --no-cpu-baseline > gpurun_out/bench_fp8.json 2> gpurun_out/bench_fp8.err
tail -c 4000 gpurun_out/bench_fp8.json; tail -5 gpurun_out/bench_fp8.err
