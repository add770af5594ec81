# round-2 re-entry baseline: GPU tests, smoke, default bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -q -m gpu --timeout 900 -x 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err; echo "bench exit $?"
tail -c 3000 gpurun_out/bench_base.json
