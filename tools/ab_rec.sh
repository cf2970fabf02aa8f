#!/bin/bash
# A/B the headline bench (ms/step) plus the recursion's phase times (F2GPU_REC_TIMES) over env settings
out=gpurun_out/abr.txt; : > $out
for e in "$@"; do
  env $e python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-gemm > gpurun_out/b.log 2>&1
  ms=$(python -c "import json; d=json.loads(open('gpurun_out/b.log').readlines()[-1]); print(d['ms_per_step'], d['parity']['status'])" 2>&1 | tail -1)
  ph=$(env $e F2GPU_REC_TIMES=1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-gemm 2>&1 | grep "\[rec\] trsm" | awk '{printf "%s %s ms; ", $2, $5}')
  echo "[$e] $ms | $ph" >> $out
done
cat $out
