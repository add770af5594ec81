# Time each prebuilt libssa variant in variants/ on the bench headline (no extra legs);
# variants named trace_* run scripts/trace_run.py instead.
set -x
mkdir -p gpurun_out
cp paper_2605_13784_b200/libssa.so /tmp/libssa_default.so
for f in variants/*.so; do
  cp $f paper_2605_13784_b200/libssa.so
  b=$(basename $f .so)
  echo "== $b"
  case $b in
    trace*) timeout 300 python scripts/trace_run.py && for k in append query; do mv gpurun_out/trace_$k.npy gpurun_out/${b}_$k.npy; mv gpurun_out/trace2_$k.npy gpurun_out/${b}_t2_$k.npy; done ;;
    *) timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --legs "${LEGS:-}" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({k:d.get(k) for k in ['append_tflops','append_tc_util','query_latency_us_per_layer','kernel_ms']}), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
        for k in ['flash_queries','multi_tenant','split_kv_128k']:
            if k in d: print(k, json.dumps(d[k]))
    else: print(l.rstrip()[:300])
" ;;
  esac
  [ -n "$PYTEST_SEL" ] && timeout 600 python -m pytest $PYTEST_SEL -q -x --timeout 300 2>&1 | tail -3
done
cp /tmp/libssa_default.so paper_2605_13784_b200/libssa.so
