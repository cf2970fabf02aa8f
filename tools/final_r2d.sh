#!/bin/bash
# round-2 final evidence (chain build): tests, bench line, phase times, traces, ncu launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r2d_gputest.log
python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
F2GPU_REC_TIMES=1 python bench.py --steps 3 --warmup 3 --no-cpu --no-gemm --no-e2e 2>&1 | grep "^\[rec\]" | tail -8 > gpurun_out/r2d_rectimes.log
python bench.py --force-dist --steps 5 --warmup 3 --no-cpu --no-gemm --no-e2e 2>/dev/null | tail -1 > gpurun_out/r2d_bench_dist.json
python tools/variants.py cfg5 > gpurun_out/r2d_variants.log 2>&1; python tools/variants.py cfg3 >> gpurun_out/r2d_variants.log 2>&1
F2GPU_GRAPHS=0 python tools/trace_leaf.py 16384 16384 100 4 > gpurun_out/r2d_trace_short.txt 2>&1
F2GPU_GRAPHS=0 python tools/trace_leaf.py 65536 4096 20 4 > gpurun_out/r2d_trace_tall.txt 2>&1
# ncu serialises kernels: k_panel_chain spins on counters of kernels launched after it, so the
# launch list is taken with the per-panel schedule (F2GPU_PANEL_CHAIN=0), everything else as shipped
F2GPU_PANEL_CHAIN=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv \
  --log-file gpurun_out/r2d_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-gemm > gpurun_out/r2d_ncu.log 2>&1
gzip -f gpurun_out/r2d_launches.csv
ls -la gpurun_out | tail -12
