#!/bin/bash
# ncu evidence for round 1: launch list of one S=20 forward + full captures of the
# global-attention FMHA and the fc1 GEMM (run from the repo root under gpurun).
set -x
CMD="python bench.py --views 20 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fmha_kernel -s 49 -c 2 -o gpurun_out/fmha $CMD > gpurun_out/ncu_fmha.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 200 -c 6 -o gpurun_out/gemm $CMD > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out
