for e in 0 1 2 3; do echo "EMU=$e"; VX_FMHA_EMU=$e timeout 300 python tools/bench_kernels.py --views 20 200 --only attn 2>&1 | grep "^attn_global"; done
