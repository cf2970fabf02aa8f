#!/bin/bash
o=gpurun_out/chain_dbg.txt; : > $o
for shape in "1024 1024" "3000 2048" "4096 4096" "8192 1024" "16384 1024"; do
  for ch in 0 1; do
    echo "== $shape chain=$ch" >> $o
    F2GPU_SPIN_DIAG=1 F2GPU_PANEL_CHAIN=$ch timeout 120 python tools/chain_dbg.py $shape 3 2>&1 | tail -4 >> $o
  done
done
cat $o
