#!/bin/bash
# Alternate FMHA configurations under sustained (power-capped) load: tools/sustain_attn.sh "VX_FMHA_EMU=2" "VX_FMHA_EMU=1" ...
for r in 1 2; do
  for c in "$@"; do
    env $c timeout 120 python tools/sustain_attn.py --label "$c" --views ${VIEWS:-200} --seconds ${SECS:-14}
  done
done
