# SURVEY §8d config 4 on one B200: views sweep (views/s, peak HBM, in-step FMHA TFLOP/s); one timed
# forward per size after one warm-up (none for >= 1500 views: minutes per forward)
for S in 50 100 500; do
  timeout 900 python bench.py --views $S --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/sweep_S$S.json
done
for S in 1500 2000; do
  timeout 2400 python bench.py --views $S --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/sweep_S$S.json
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/sweep_S*.json"), key=lambda x: int(x.split("_S")[1].split(".")[0])):
    try:
        d = json.load(open(f))
        print(d["config"]["views"], round(d["value"], 3), round(d["ms_per_step"], 1), round(d["peak_hbm_gb_per_gpu"], 2),
              round(d["roofline"]["achieved"], 1), d["clocks"]["sm_mhz"])
    except Exception as e:
        print(f, "failed", e)
PY
