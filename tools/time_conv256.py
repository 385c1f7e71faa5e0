import sys, runpy, torch
sys.argv = ["prof_layer.py", "conv256", "200"]
g = runpy.run_path("tools/prof_layer.py")
run = g["run"]
for _ in range(3): run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): run()
e.record(); e.synchronize()
ms = s.elapsed_time(e) / 20
fl = 2 * 16 * 148 * 148 * 256 * 2304
print(f"conv256 16x148^2: {ms:.3f} ms, {fl / ms / 1e9:.0f} TFLOP/s")
