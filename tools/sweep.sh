#!/bin/bash
# quick SpMM schedule sweep on the GPU box: prints ms_per_step / GFLOP/s / frac
# usage: tools/sweep.sh TB:W[:RING] ...
for cfg in "$@"; do
  IFS=: read tb w ring <<< "$cfg"
  SPX_SPMM_RING=${ring:-8} timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 0 --tb $tb --warp $w 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['value'], d['roofline']['frac'])" || echo "$cfg FAILED"
done
