# FMHA 4x48 ones-column (SUMV) variant: EMU sweep + frame/global comparison vs the 4x64 / 3x64 kernels
for e in 1 2 3 4; do echo "CFG=5 EMU=$e"; VX_FMHA_CFG=5 VX_FMHA_EMU=$e timeout 300 python tools/bench_kernels.py --views 20 200 --only attn 2>&1 | grep "^attn_"; done
echo "default"; timeout 300 python tools/bench_kernels.py --views 20 200 --only attn 2>&1 | grep "^attn_\|^sdpa"
