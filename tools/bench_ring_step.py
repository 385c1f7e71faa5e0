"""Time one ring step of frame-sharded global attention (vx_attention_merge, mode 2) on one GPU, alone and
with the ring's K/V transfer running concurrently.

Shape of rank r's step at S views over g ranks: Lq = Lk = (S/g) * 1374 tokens, 16 heads, d=64.  The
concurrent transfer is a real NCCL send/recv of the step's packed K/V block (2 * 16 * Lk * 64 bf16,
140 MB at S=200, g=8) through a world-size-1 process group (rank 0 sends to itself), issued exactly as
ring.TorchDistComm does before the step's FMHA: its kernel takes SMs while the persistent FMHA grid
starts.  Reports ms per step alone, NCCL alone, step + concurrent NCCL, and the overhead.

A/B against static round-robin units: VX_LIB=exp/libvx_diag.so VX_FMHA_STATIC=1 (diagnostic build,
paper_2509_25191_b200.build.build_diag).  With the diagnostic build, --hog K also measures the step
with K SMs held for --hog-us microseconds by a kernel launched just before it (512 threads and 120 KB
of shared memory per CTA, so no FMHA CTA fits next to it): an NCCL transfer kernel that keeps its SMs
for the transfer's duration, which the world-size-1 self send/recv above may not (it can take the copy
engine).
"""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--hog", type=int, nargs="*", default=[])
    ap.add_argument("--hog-us", type=float, default=300.0)
    ap.add_argument("--hog-first", type=float, default=0.0, help="host delay (us) between the hog and the FMHA launch")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2509_25191_b200 import ops
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    H, d = 16, 64
    res = {}

    def timed(fn, reps):
        ts = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        return ts[len(ts) // 2]  # median

    for g in args.ranks:
        T = (args.views // g) * 1374
        q, k, v = (torch.randn(H, T, d, device="cuda").bfloat16() for _ in range(3))
        o_acc = torch.zeros(T, H * d, device="cuda")
        lse = torch.zeros(H, T, device="cuda")
        blk = torch.empty(2, H, T, d, device="cuda", dtype=torch.bfloat16)
        rcv = torch.empty_like(blk)

        def step():
            ops.attention_merge(q, k, v, 2, o_acc, lse, Lq=T, Lk=T)

        def xfer():
            return dist.batch_isend_irecv([dist.P2POp(dist.isend, blk, 0), dist.P2POp(dist.irecv, rcv, 0)])

        def xfer_only():
            for r in xfer():
                r.wait()

        def step_with_xfer():
            reqs = xfer()
            step()
            for r in reqs:
                r.wait()

        for f in (step, xfer_only, step_with_xfer):
            for _ in range(3):
                f()
        torch.cuda.synchronize()
        t_step = timed(step, args.reps)
        t_x = timed(xfer_only, args.reps)
        t_both = timed(step_with_xfer, args.reps)
        res[f"g{g}"] = {"tokens": T, "block_mb": round(blk.numel() * 2 / 1e6, 1), "step_ms": round(t_step, 3),
                        "nccl_ms": round(t_x, 3), "step_with_nccl_ms": round(t_both, 3),
                        "overhead_pct": round(100 * (t_both / t_step - 1), 2),
                        "tflops": round(4.0 * H * T * T * d / t_step / 1e9, 1)}
        if args.hog:
            import ctypes
            lib = ops.load_library() if ops._lib is None else ops._lib
            if not hasattr(lib, "vx_diag_sm_hog"):
                raise SystemExit("--hog needs the diagnostic library (VX_LIB=exp/libvx_diag.so)")
            lib.vx_diag_sm_hog.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_int, ctypes.c_void_p]
            hog_stream = torch.cuda.Stream()
            cycles = int(args.hog_us * 1e-6 * 1.9e9)
            for nh in args.hog:
                def step_with_hog():
                    """FMHA step launched while `nh` SMs are held (the hog is resident first); timed from the
                    FMHA launch to the later of the step's and the hog's end."""
                    hog_stream.wait_stream(torch.cuda.current_stream())
                    assert lib.vx_diag_sm_hog(nh, cycles, 120 * 1024, ctypes.c_void_p(hog_stream.cuda_stream)) == 0
                    time.sleep(args.hog_first * 1e-6)
                    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s_.record()
                    step()
                    torch.cuda.current_stream().wait_stream(hog_stream)
                    e_.record()
                    e_.synchronize()
                    return s_.elapsed_time(e_)

                # alternate dynamic / static units (diagnostic build: VX_FMHA_STATIC read per launch) and the
                # undisturbed step, so clock drift hits all three alike
                ts = {"alone": [], "dynamic": [], "static": []}
                for _ in range(args.reps):
                    for mode in ("alone", "dynamic", "static"):
                        os.environ["VX_FMHA_STATIC"] = "1" if mode == "static" else "0"
                        torch.cuda.synchronize()
                        if mode == "alone":
                            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            s_.record()
                            step()
                            e_.record()
                            e_.synchronize()
                            ts[mode].append(s_.elapsed_time(e_))
                        else:
                            ts[mode].append(step_with_hog())
                os.environ["VX_FMHA_STATIC"] = "0"
                med = {k: sorted(v)[len(v) // 2] for k, v in ts.items()}
                res[f"g{g}"][f"hog{nh}"] = {k: round(v, 3) for k, v in med.items()}
                res[f"g{g}"][f"hog{nh}"].update({f"{k}_overhead_pct": round(100 * (med[k] / med["alone"] - 1), 2)
                                                  for k in ("dynamic", "static")})
    sched = "static" if os.environ.get("VX_FMHA_STATIC") == "1" else "dynamic"  # of the NCCL rows
    print(json.dumps({"sched": sched, "views": args.views, "hog_us": args.hog_us if args.hog else None,
                      "hog_first_us": args.hog_first, **res}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
