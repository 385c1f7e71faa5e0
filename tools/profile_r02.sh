#!/bin/bash
# ncu evidence for round 2 (repo root, one GPU, under gpurun): the S=20 forward's launch list (bench
# command, cold-cache serialised times) and full captures of the S=200 layer kernels.
CMD="python bench.py --views 20 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
NCU=/usr/local/cuda/bin/ncu
$CMD > gpurun_out/plain.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_S20.csv $CMD \
  > gpurun_out/ncu_launches.log 2>&1
for w in attn_global attn_frame proj fc2 qkv; do
  case $w in attn_*) K=fmha_kernel;; *) K=gemm_kernel;; esac
  python tools/prof_layer.py $w 200 > gpurun_out/plain_$w.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/r02_${w}_S200 \
    python tools/prof_layer.py $w 200 > gpurun_out/ncu_$w.log 2>&1
  echo "$w rc=$?"
done
ls -la gpurun_out | grep -E "ncu-rep|csv"
