#!/bin/bash
# stability of the chain build: the GPU suite 3x, the bench (with e2e) 4x, 10 rounds of dbg_repeat,
# the full-size digest file 2x more, smoke
o=gpurun_out/r2d_stress.txt; : > $o
for i in 1 2 3; do timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1 >> $o; done
for i in 1 2 3 4; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-gemm 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['parity']['status'], d['e2e']['ms_per_step'], d['e2e']['parity'])" >> $o 2>&1; done
timeout 900 python tools/dbg_repeat.py 10 2>&1 | tail -2 >> $o
for i in 1 2; do timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -1 >> $o; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $o 2>&1
timeout 600 python bench.py --force-dist --steps 5 --warmup 3 --no-cpu --no-gemm --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('dist', d['ms_per_step'], d['parity']['status'])" >> $o 2>&1
timeout 600 python bench.py --variant block --steps 5 --warmup 3 --no-cpu --no-gemm 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('block', d['ms_per_step'], d['parity']['status'], d['e2e']['ms_per_step'], d['e2e']['parity'])" >> $o 2>&1
cat $o
