#!/bin/bash
# A/B the headline bench (ms/step) over env settings given as arguments
out=gpurun_out/abb.txt; : > $out
for e in "$@"; do
  env $e python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-gemm > gpurun_out/b.log 2>&1
  ms=$(python -c "import json; d=json.loads(open('gpurun_out/b.log').readlines()[-1]); print(d['ms_per_step'])" 2>&1 | tail -1)
  echo "[$e] $ms" >> $out
done
cat $out
