#!/bin/bash
# round-2 follow-up captures (repo root, one GPU, under gpurun): the steady-state launch list of the S=20
# bench (NVTX range "timed_steps" only) and a full capture of the TMA-epilogue proj GEMM at S=200.
NCU=/usr/local/cuda/bin/ncu
CMD="python bench.py --views 20 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_ss.log 2>&1 && \
$NCU --nvtx --nvtx-include "timed_steps/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_S20_steady.csv $CMD > gpurun_out/ncu_launches_ss.log 2>&1
echo "steady launches rc=$?"
python tools/prof_layer.py proj 200 > gpurun_out/plain_proj2.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/r02_proj_tma_S200 \
  python tools/prof_layer.py proj 200 > gpurun_out/ncu_proj2.log 2>&1
echo "proj rc=$?"
ls -la gpurun_out | grep -E "steady|proj_tma"
