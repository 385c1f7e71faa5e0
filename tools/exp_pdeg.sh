for e in 2 3; do
 echo "deg3 EMU=$e"; VX_FMHA_EMU=$e timeout 200 python tools/bench_kernels.py --views 20 200 --only attn 2>&1 | grep "^attn_global"
 echo "deg2 EMU=$e"; VX_LIB=$PWD/exp/libvx_deg2.so VX_FMHA_EMU=$e timeout 200 python tools/bench_kernels.py --views 20 200 --only attn 2>&1 | grep "^attn_global"
done
VX_LIB=$PWD/exp/libvx_deg2.so timeout 200 python -m pytest tests/test_kernels_gpu.py -m gpu -q -k attention 2>&1 | tail -1
