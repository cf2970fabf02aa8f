#!/bin/bash
# A/B the headline bench + the 16384^2 leaf over env settings given as arguments:
#   tools/ab.sh "F2GPU_X=1" "F2GPU_X=0 F2GPU_Y=1" ...
out=gpurun_out/ab.txt; : > $out
for e in "$@"; do
  env $e python bench.py --steps 5 --warmup 3 > gpurun_out/b.log 2>&1
  ms=$(python -c "import json; d=json.loads(open('gpurun_out/b.log').readlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])" 2>&1 | tail -1)
  leaf=$(env $e python tools/leaf_bench.py 16384 16384 2>&1 | tail -1)
  echo "[$e] bench $ms leaf16k $leaf" >> $out
done
cat $out
