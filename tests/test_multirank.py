"""Multi-process runs on one GPU through the real torch.distributed API (gloo; the exchange is staged
through host memory because NCCL needs one GPU per rank): the sharded forward via ring.TorchDistComm
under torch.distributed.run, and bench.py's multi-rank flow (--gpus N self-launch, barriers,
max-over-ranks timing, end-to-end leg).  The NCCL transport itself needs one GPU per rank."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,views", [(2, 5), (3, 7)])
def test_torchrun_sharded_forward_gloo(tmp_path, world, views):
    out = str(tmp_path / "res")
    env = dict(os.environ, OUT=out, VIEWS=str(views))
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "dist_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = [json.load(open(f"{out}.{i}")) for i in range(world)]
    for x in res:
        assert x["frame_offset"] == x["lo"]
        for k in ("depth", "depth_conf", "world_points", "world_points_conf"):
            assert x[k] < 1e-2, x
        assert x["pose_vs_single"] < 1e-2
        assert x["pose"] == res[0]["pose"]  # pose_enc bit-identical on every rank


def test_bench_two_ranks_gloo():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo", "--views", "4",
           "--steps", "1", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "2 ranks" in d["config"]["parallelism"]
