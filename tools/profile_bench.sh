#!/bin/bash
# Run on the GPU box: launch list of the bench step + one full ncu capture of
# the dominant kernel (the A*G DMMA GEMM). Outputs under gpurun_out/.
set -e
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-secondary"
$CMD > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/prof_ncu_list.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:dgemm_kernel -s 0 -c 1 -o gpurun_out/prof_dgemm_full $CMD > gpurun_out/prof_ncu_full.log 2>&1
echo done
