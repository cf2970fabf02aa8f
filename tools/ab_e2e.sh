#!/bin/bash
# A/B the e2e (host-buffer) leg of bench.py over env settings given as arguments
out=gpurun_out/abe.txt; : > $out
for e in "$@"; do
  env $e python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/b.log 2>&1
  r=$(python -c "import json; d=json.loads(open('gpurun_out/b.log').readlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'])" 2>&1 | tail -1)
  echo "[$e] device/e2e ms $r" >> $out
done
cat $out
