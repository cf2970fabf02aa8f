#!/bin/bash
# A/B of the persistent panel-chain kernel (F2GPU_PANEL_CHAIN=1): parity, leaf timings, trace, bench
o=gpurun_out/chain_ab.txt; : > $o
echo "== parity (chain)" >> $o
F2GPU_PANEL_CHAIN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "decompose" 2>&1 | tail -5 >> $o
for shape in "16384 16384" "32768 8192" "65536 4096"; do
  for ch in 0 1; do
    echo "== leaf $shape chain=$ch" >> $o
    F2GPU_PANEL_CHAIN=$ch timeout 300 python tools/leaf_bench.py $shape 2>&1 | tail -1 >> $o
  done
done
echo "== trace chain=1 16384x16384" >> $o
F2GPU_PANEL_CHAIN=1 timeout 300 python tools/trace_leaf.py 16384 16384 2>&1 | tail -30 >> $o
echo "== trace chain=1 65536x4096" >> $o
F2GPU_PANEL_CHAIN=1 timeout 300 python tools/trace_leaf.py 65536 4096 2>&1 | tail -30 >> $o
echo "== bench" >> $o
for e in "F2GPU_PANEL_CHAIN=0" "F2GPU_PANEL_CHAIN=1" "F2GPU_PANEL_CHAIN=1 F2GPU_CHAIN_SMS=1"; do
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-gemm > gpurun_out/b.log 2>&1
  echo "[$e] $(python -c "import json; d=json.loads(open('gpurun_out/b.log').readlines()[-1]); print(d['ms_per_step'], d['parity']['status'])" 2>&1 | tail -1)" >> $o
done
cat $o
