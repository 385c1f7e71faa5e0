#!/bin/bash
# correctness + timing of the FMHA for several FMA-pipe exp fractions (VX_FMHA_EMU pairs of 8)
for e in ${EMUS:-0 2 3 4}; do
  echo "== EMU=$e"
  VX_FMHA_EMU=$e timeout 120 python tools/dbg_attn.py 2>&1 | tail -6
  VX_FMHA_EMU=$e timeout 200 python tools/bench_kernels.py --views ${VIEWS:-20} --only attn 2>&1 | grep "attn_\|sdpa_"
done
