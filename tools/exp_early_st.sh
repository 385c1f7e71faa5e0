# FMHA: early partial P store (first 16 columns while the last 8 exp pairs run) vs the previous build
timeout 200 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k attention --timeout 60 2>&1 | tail -1
timeout 200 python tools/bench_kernels.py --views 20 200 --only attn 2>&1 | grep "^attn_"
VX_LIB=$PWD/exp/libvx_prev.so timeout 200 python tools/bench_kernels.py --views 20 200 --only attn 2>&1 | grep "^attn_"
