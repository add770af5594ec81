for r in 1 2 3; do
  AB_ONLY_DEFAULT=1 python scripts/ab_step.py 2>&1 | grep AB | head -1 | sed "s/^/cur /"
  AB_ONLY_DEFAULT=1 python variants/r1/scripts/ab_step.py 2>&1 | grep AB | head -1 | sed "s/^/r1 /"
done
