#!/bin/bash
# correctness + timing of the FMHA for several FMA-pipe exp fractions / polynomial degrees
for cfg in ${CFGS:-"2 3"}; do
  set -- $cfg
  echo "== EMU=$1 PDEG=$2"
  VX_FMHA_EMU=$1 VX_FMHA_PDEG=$2 timeout 120 python tools/dbg_attn.py 2>&1 | tail -6 | head -2
  VX_FMHA_EMU=$1 VX_FMHA_PDEG=$2 timeout 200 python tools/bench_kernels.py --views ${VIEWS:-20} --only attn 2>&1 | grep "attn_"
done
