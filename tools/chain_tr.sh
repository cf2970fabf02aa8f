#!/bin/bash
o=gpurun_out/chain_tr.txt; : > $o
for shape in "16384 16384" "65536 4096"; do
echo "== trace chain=1 $shape" >> $o
F2GPU_PANEL_CHAIN=1 timeout 300 python tools/trace_leaf.py $shape 100 6 2>&1 | tail -45 >> $o
done
cat $o
