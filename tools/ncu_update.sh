#!/bin/bash
# ncu --set full capture of one north-star update launch (k_update_v3 or _v4 per F2GPU_UPDATE)
# usage: tools/ncu_update.sh OUTNAME [regex]
out=${1:-upd}; rx=${2:-k_update_v}
ncu --set full --import-source on --clock-control none -k regex:$rx -s 1 -c 1 -o gpurun_out/$out -f \
  python tools/prof_kernels.py update > gpurun_out/$out.log 2>&1
ncu -i gpurun_out/$out.ncu-rep --page raw --csv > gpurun_out/$out.raw.csv 2>/dev/null
ncu -i gpurun_out/$out.ncu-rep --page source --csv --print-source sass > gpurun_out/$out.src.csv 2>/dev/null
echo "ncu rc done"
