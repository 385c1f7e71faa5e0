# GA optimiser timing at 200 views (tools/bench_ga.py); the pair-kernel shape sweep that picked
# GA_PAIR_THREADS/UNROLL in csrc/ga.cu was run with a VX_GA_PAIR switch since removed:
#   256 thr x1: 182 us/eval, 128x2: 144, 256x2: 143, 128x4: 119, 128x8: 118, 64x4: 119
timeout 300 python tools/bench_ga.py --no-cpu --repeats 1 2>&1 | tail -1
