# A/B of two library builds on the GEMM kernel bench (exp/libvx_base.so vs exp/libvx_pre.so), interleaved
for i in 1 2; do
  for l in base pre; do echo "$l"; VX_LIB=$PWD/exp/libvx_$l.so timeout 200 python tools/bench_kernels.py --views 200 --only gemm 2>&1 | grep "^gemm_" | grep -v nogelu; done
done
