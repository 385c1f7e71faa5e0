#!/bin/bash
# ncu evidence for the current kernels (run from the repo root under gpurun, one GPU):
#   launch list of one S=20 forward (same command as bench, cold-cache serialised times);
#   full capture of one S=20 global-attention launch (tools/prof_attn.py, the 2nd launch);
#   DRAM traffic of one S=200 global-attention launch (for bench.py's roofline.traffic).
set -x
CMD="python bench.py --views 20 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
python tools/prof_attn.py 20 > gpurun_out/plain_attn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fmha_kernel -s 1 -c 1 -o gpurun_out/fmha_final python tools/prof_attn.py 20 > gpurun_out/ncu_fmha.log 2>&1
python tools/prof_attn.py 200 > gpurun_out/plain_a200.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fmha_kernel -s 1 -c 1 --csv --log-file gpurun_out/fmha_S200_traffic.csv python tools/prof_attn.py 200 > gpurun_out/ncu_a200.log 2>&1
ls -la gpurun_out | tail -20
# full capture of one CTA-pair GEMM launch (fc1 + GELU at the S=20 shape, via the kernel bench)
python tools/bench_kernels.py --views 20 --only gemm > gpurun_out/plain_gemm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 1 -o gpurun_out/gemm_cg2 python tools/bench_kernels.py --views 20 --only gemm > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out | tail -5
