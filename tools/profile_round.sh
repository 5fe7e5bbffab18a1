#!/bin/bash
# Run on the GPU box (one GPU): the launch list of the bench step and one full
# ncu capture each of the dominant kernels (A*G DMMA GEMM, batched 32x32, the
# real-input FFT circulant kernel, the device Gaussian generator, a GENP panel,
# the overlap-save Toeplitz kernel). Each command
# first runs once without ncu. Outputs under gpurun_out/prof/.
set -e
mkdir -p gpurun_out/prof
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-secondary --no-configs"
$CMD > gpurun_out/prof/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_bench.csv $CMD > gpurun_out/prof/ncu_list.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:dgemm_kernel -s 0 -c 1 -o gpurun_out/prof/dgemm $CMD > gpurun_out/prof/ncu_dgemm.log 2>&1
python tools/time_batched.py > gpurun_out/prof/batched_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:batched_genp32 -c 1 -o gpurun_out/prof/batched python tools/time_batched.py > gpurun_out/prof/ncu_batched.log 2>&1
python tools/run_circ.py > gpurun_out/prof/circ_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:rows_kernel -c 1 -o gpurun_out/prof/fft_rows python tools/run_circ.py > gpurun_out/prof/ncu_fft.log 2>&1
python tools/run_gen.py > gpurun_out/prof/gen_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gen_kernel -c 1 -o gpurun_out/prof/gen python tools/run_gen.py > gpurun_out/prof/ncu_gen.log 2>&1
python tools/run_genp.py > gpurun_out/prof/genp_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:lu_panel64 -s 100 -c 1 -o gpurun_out/prof/panel python tools/run_genp.py > gpurun_out/prof/ncu_panel.log 2>&1
python tools/time_toep.py > gpurun_out/prof/toep_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:ola_rows -s 1 -c 1 -o gpurun_out/prof/ola_rows python tools/time_toep.py > gpurun_out/prof/ncu_ola.log 2>&1
echo done
