"""Is the heads phase host-bound? Times, at S views, the host time to issue the three heads (no
sync) against their device time, and the heads phase inside a full forward.

    python tools/heads_host_probe.py [S]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_25191_b200 import profiling  # noqa: E402
from paper_2509_25191_b200.config import vggt_1b  # noqa: E402
from paper_2509_25191_b200.heads import camera_head  # noqa: E402
from paper_2509_25191_b200.vggt import VGGT  # noqa: E402
from paper_2509_25191_b200.weights import make_state_dict, synthetic_images  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = vggt_1b()
m = VGGT(cfg, state_dict=make_state_dict(cfg, 0))
imgs = synthetic_images(cfg, S, 1).cuda()
with torch.no_grad():
    m(imgs)
    torch.cuda.synchronize()
    t = profiling.PhaseTimer()
    profiling.set_timer(t)
    t0 = time.perf_counter()
    m(imgs)
    th = time.perf_counter() - t0
    torch.cuda.synchronize()
    tw = time.perf_counter() - t0
    profiling.set_timer(None)
    ph = t.summary()
    print(f"forward: host issue {th * 1e3:.1f} ms, wall {tw * 1e3:.1f} ms; phases "
          + ", ".join(f"{k} {v['total_ms']:.2f}" for k, v in ph.items()), flush=True)

    local, f0, _ = m._local(imgs, False)
    kept = m._aggregate(local, f0)
    cam = kept[cfg.kept_layers[-1]][:, 0]
    H = W = cfg.img_size
    depth = torch.empty(S, H, W, 1, device="cuda")
    dconf = torch.empty(S, H, W, device="cuda")
    pts = torch.empty(S, H, W, 3, device="cuda")
    pconf = torch.empty(S, H, W, device="cuda")
    s_d, s_p = m._head_streams(torch.device("cuda"))
    for name, fn in [("depth head", lambda: m.depth_head(kept, depth, dconf, cfg.head_chunk)),
                     ("point head", lambda: m.point_head(kept, pts, pconf, cfg.head_chunk)),
                     ("camera head", lambda: camera_head(m.W, cam))]:
        for rep in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # queue a long device op first so the host issue time is not hidden behind an idle GPU
            e0.record()
            t0 = time.perf_counter()
            fn()
            th = time.perf_counter() - t0
            e1.record()
            torch.cuda.synchronize()
            tw = time.perf_counter() - t0
        print(f"{name}: host issue {th * 1e3:.2f} ms, device {e0.elapsed_time(e1):.2f} ms, wall {tw * 1e3:.2f} ms",
              flush=True)

    # device kernels of one depth-head call (CUPTI via torch.profiler): busy time vs span
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        m.depth_head(kept, depth, dconf, cfg.head_chunk)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    busy = sum(e.device_time for e in evs) / 1e3
    span = (max(e.time_range.end for e in evs) - min(e.time_range.start for e in evs)) / 1e3
    print(f"depth head kernels: {len(evs)} launches, busy {busy:.2f} ms, span {span:.2f} ms", flush=True)
    agg = {}
    for e in evs:
        a = agg.setdefault(e.name[:70], [0, 0.0])
        a[0] += 1
        a[1] += e.device_time / 1e3
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
        print(f"  {ms:7.3f} ms {n:4d}  {k}")
    print("first chunk, in launch order:")
    for e in sorted(evs, key=lambda e: e.time_range.start)[:42]:
        print(f"  {e.device_time:8.1f} us  {e.name[:60]}")
