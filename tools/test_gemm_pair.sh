# CTA-pair (cta_group::2) GEMM: correctness under a hard timeout (all GPU tests), then speed
export VX_GEMM_PAIR=2
timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -3
timeout 120 python tools/bench_kernels.py --views 20 200 --only gemm 2>&1 | grep "^gemm_"
timeout 300 python bench.py --views 20 --steps 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S20', d['value'], d['phases_ms_per_step'])"
export VX_GEMM_PAIR=1
timeout 300 python bench.py --views 20 --steps 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S20 mc', d['value'], d['phases_ms_per_step'])"
