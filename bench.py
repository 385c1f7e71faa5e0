"""Benchmark of the dense-view VGGT inference path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--views S] [--impl vx|reference]

One step = one full VGGT forward (aggregator 24x2 blocks + camera head + both
DPT heads, frame-chunked) of S views at 518x518 on the VGGT-1B-shaped model
with seeded random-init weights (no checkpoints exist offline) and synthetic
torch.rand images.  Default workload: S = 200 views ("views/sec at 200
views"), BASELINE.json configs[2].  Under torchrun (N > 1) the same S views are
frame-sharded over the ranks (global attention K/V ring): strong scaling.

`value` is device-timed with CUDA events (images already in HBM, max over
ranks); `e2e` runs the public API from pinned host images to host outputs with
the copies inside the timed region.  `--impl reference` times the CPU oracle
(this repo's fp32 restatement; the reference ships no implementation of this
path) on a bounded sample and reports the same metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "VGGT views/sec at 200 & 1000 views (1/2/4/8 B200); peak HBM/GPU; MMA util"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


def self_launch(args) -> None:
    """`bench.py --gpus N` outside torchrun: re-exec this command under torch.distributed.run with N
    ranks (one process per GPU, rendezvous on 127.0.0.1); fail loudly if fewer than N GPUs exist."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return  # the reference arm runs on rank 0's host cores only: nothing to launch
    n = torch.cuda.device_count()
    if n < args.gpus and args.dist_backend == "nccl":
        raise SystemExit(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n}")
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------
def cpu_oracle_sample(cfg, sd, S_target, threads=None):
    """The fp32 CPU oracle timed per work unit at the S-view shapes and composed into an S-view forward
    (oracle/cpu_baseline.py); the composition's error against directly measured forwards / global
    blocks on the same kind of host (tools/cpu_baseline_check.py) is attached when it was recorded."""
    from oracle.cpu_baseline import cpu_baseline
    r = cpu_baseline(cfg, sd, S_target, threads=threads)
    chk = os.path.join(ROOT, "profiles", "r02_cpu_baseline_check.json")
    if os.path.exists(chk):
        with open(chk) as f:
            c = json.load(f)
        r["composition_check"] = {"threads": c.get("threads"),
                                  "checks": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in x.items()
                                              if k != "units_s"} for x in c["checks"]]}
    r["measured_s"] = r.pop("sample_wall_s")
    return r


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2509_25191_b200.config import vggt_1b
    from paper_2509_25191_b200.weights import make_state_dict
    cfg = vggt_1b()
    sd = make_state_dict(cfg, 0)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg, sd, args.views, threads=threads)
    vals, secs, fwd, r = [], [], [], None
    for _ in range(args.steps):
        r = cpu_oracle_sample(cfg, sd, args.views, threads=threads)
        vals.append(r["value"])
        secs.append(r["measured_s"])  # wall time of the step's bounded sample
        fwd.append(r["forward_s"])    # the composed S-view forward it measures
    v = statistics.median(vals)
    cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
    cpu["value"] = v
    if "composition_check" in r:
        cpu["composition_check"] = r["composition_check"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "views/s", "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (torch.rand views seed 1, random-init weights seed 0)",
        "config": {"workload": f"vggt1b_518_S{args.views}", "views": args.views, "img": 518,
                   "tokens_per_view": cfg.tokens_per_frame, "model": "VGGT-1B-shaped (24x2 blocks, C=1024)",
                   "parallelism": "CPU host cores (rank 0 only)",
                   "l2": "n/a (CPU oracle; each step times every work unit of the S-view forward at its S-view "
                         "shape on a bounded slice and composes the forward, see cpu_baseline.sample)"},
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "composed_forward_s": statistics.median(fwd),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,memory.used")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, mx, reasons, mem, pw = [], 0.0, set(), [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                pw.append(float(r[2]))
                for n, v in zip(names, r[3:7]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(n)
                mem.append(float(r[7]))
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if pw:
            out["power_w_median"] = statistics.median(pw)
        if mem:  # device memory in use (whole process incl. context, NCCL and the allocator's cache), MiB
            out["memory_used_gb_max"] = round(max(mem) * 1.048576e-3, 2)
        return out


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--impl", default="vx", choices=["vx", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-heads", action="store_true", help="aggregator only (diagnostic)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: ranks may share GPUs and the ring exchange is staged through host memory "
                         "(tests the multi-rank flow on one GPU; not a performance configuration)")
    ap.add_argument("--patch-embed", default="conv", choices=["conv", "dinov2"],
                    help="conv (the north star's patch-embed GEMM, default) or the DINOv2 encoder of released checkpoints")
    args = ap.parse_args()
    self_launch(args)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    if args.impl == "reference":
        return run_reference(args)

    import torch.distributed as dist
    from paper_2509_25191_b200 import ops, profiling
    from paper_2509_25191_b200.config import vggt_1b
    from paper_2509_25191_b200.vggt import VGGT
    from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
    from oracle.vggt_ref import forward_flops

    world, rank, local = dist_env()
    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    cfg = vggt_1b().with_(patch_embed=args.patch_embed)
    S = args.views
    sd = make_state_dict(cfg, 0)
    model = VGGT(cfg, state_dict=sd, dist=world > 1)
    images = synthetic_images(cfg, S, seed=1)
    images_dev = images.cuda()
    peaks = load_peaks()

    def step(x):
        if args.no_heads:
            return model.aggregator(x)
        return model(x)

    for _ in range(args.warmup):
        step(images_dev)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()

    timer = profiling.PhaseTimer()
    profiling.set_timer(timer)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ops.kernel_launches()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    torch.cuda.nvtx.range_push("timed_steps")  # ncu --nvtx --nvtx-include "timed_steps/": steady-state launches
    for _ in range(args.steps):
        step(images_dev)
    torch.cuda.nvtx.range_pop()
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    profiling.set_timer(None)
    launches = (ops.kernel_launches() - launches0) // args.steps
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = tt.item()
    peak_hbm = torch.cuda.max_memory_allocated() / 1e9
    phases = timer.summary()
    ms_per_step = ms / args.steps
    value = S * args.steps / (ms / 1000.0)

    # roofline of the dominant kernel: global-attention FMHA (4 T^2 C FLOP per launch on 1 GPU;
    # per rank 4 T_local T C with the ring)
    N = cfg.tokens_per_frame
    T = S * N
    T_local = T // world
    attn_flops = 4.0 * T_local * T * cfg.embed_dim
    ga = phases.get("attn_global")
    roofline = None
    if ga:
        # per global layer: one launch on one GPU, the g ring steps with frame sharding, or (above
        # cfg.q_chunk views) one launch per chunk of queries — all of a layer's time / layers
        layer_ms = ga["total_ms"] / (args.steps * cfg.depth)
        achieved = attn_flops / (layer_ms / 1000.0) / 1e12
        peak = peaks["bf16_tflops_sustained"]
        traffic = None
        tp = os.path.join(ROOT, "profiles", "fmha_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("views") == S:  # measured for this workload's launch only
                traffic = tj.get("dram_bytes_per_launch")
        roofline = {"bound": "tensor", "kernel": "vx fmha_kernel<64> global attention (max-free launch + exact-fixup check launch; per layer: one launch, or one per query chunk above cfg.q_chunk views)",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "peak_source": peaks["source"] + " bf16_tflops_sustained",
                    "flops_per_launch": attn_flops, "avg_launch_ms": layer_ms, "traffic": traffic}
    total_flops = forward_flops(cfg, S, with_heads=not args.no_heads) / world
    model_tflops = total_flops / (ms_per_step / 1000.0) / 1e12

    # ---- end to end through the public API: pinned host images -> host outputs
    e2e = None
    if not args.no_e2e:
        host = images.pin_memory()
        outs = None
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        d2h = 0
        keys = ["pose_enc", "depth", "depth_conf", "world_points", "world_points_conf"]
        # a serving loop: each step's outputs go to pinned host memory on a copy stream while the
        # next step (whose own H2D copy is part of model(host)) already runs
        copy_stream = torch.cuda.Stream()
        for it in range(args.steps + 1):
            if it <= 1:  # untimed first step, then align the ranks once before the timed steps
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
            if it == 1:
                e0.record()
            out = model(host)  # each rank copies only its frames (VGGT._local slices the host batch)
            if outs is None:
                outs = {k: torch.empty(out[k].shape, dtype=out[k].dtype, pin_memory=True) for k in keys}
                d2h = sum(v.numel() * v.element_size() for v in outs.values())
                h2d = out["images"].numel() * 4
            copy_stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(copy_stream):
                for k in keys:
                    outs[k].copy_(out[k], non_blocking=True)
                    out[k].record_stream(copy_stream)
            del out
        torch.cuda.current_stream().wait_stream(copy_stream)
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ems], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = tt.item()
            nb = torch.tensor([h2d, d2h], device="cuda", dtype=torch.float64)  # whole-job bytes
            dist.all_reduce(nb, op=dist.ReduceOp.SUM)
            h2d, d2h = int(nb[0].item()), int(nb[1].item())
        e2e = {"value": S * args.steps / (ems / 1000.0), "unit": "views/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        del images_dev
        cpu = cpu_oracle_sample(cfg, sd, S)
        for k in ("measured_s", "units_s", "forward_s"):
            cpu.pop(k, None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (torch.rand views seed 1, random-init weights seed 0)",
            "config": {"workload": f"vggt1b_518_S{S}" + ("_dinov2" if args.patch_embed == "dinov2" else "")
                       + ("_aggregator_only" if args.no_heads else ""),
                       "views": S, "img": 518, "tokens_per_view": N, "model": "VGGT-1B-shaped (24x2 blocks, C=1024)",
                       "parallelism": (f"frame-sharded ring over {world} ranks ({args.dist_backend})" if world > 1
                                       else "single GPU"),
                       "l2": f"inputs larger than L2 (views {S * 3 * 518 * 518 * 4 / 1e6:.0f} MB fp32, weights "
                             f"1.8 GB bf16, both read every step; L2 126 MB)"},
            "peak_hbm_gb_per_gpu": peak_hbm,
            "model_tflops_per_gpu": model_tflops,
            "model_frac_of_peak": model_tflops / peaks["bf16_tflops_sustained"],
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "phases_ms_per_step": {k: round(v["total_ms"] / args.steps, 3) for k, v in phases.items()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
