# A/B of library variants on the bench step: interleaved single-setting runs per variant, 3 rounds.
cp paper_2605_13784_b200/libssa.so /tmp/libssa_base.so
for r in 1 2 3; do
  for v in base "$@"; do
    if [ $v = base ]; then cp /tmp/libssa_base.so paper_2605_13784_b200/libssa.so; else cp variants/$v/libssa.so paper_2605_13784_b200/libssa.so; fi
    AB_ONLY_DEFAULT=1 python scripts/ab_step.py 2>&1 | grep AB | head -1 | sed "s/^/$v /"
  done
done
cp /tmp/libssa_base.so paper_2605_13784_b200/libssa.so
