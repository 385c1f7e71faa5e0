# FMHA: default (try_wait without the suspend-time hint on the P-ready / S-ready waits) vs CFG=14 (10 ms hint)
VX_FMHA_CFG=14 timeout 200 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k attention --timeout 60 2>&1 | tail -1
for c in 0 14 0 14; do echo "CFG=$c"; VX_FMHA_CFG=$c timeout 200 python tools/bench_kernels.py --views 20 200 --only attn 2>&1 | grep "^attn_global"; done
