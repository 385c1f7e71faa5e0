"""Drop-in `VGGT` inference module (SURVEY.md §8b "Python API to keep").

    model = VGGT(cfg)                 # seeded random-init weights (no checkpoints on disk)
    preds = model(images)             # images (S,3,H,W) or (B,S,3,H,W) in [0, 1] (B scenes run in turn)
    preds["pose_enc"]                 # (1, S, 9) fp32  [T(3), quat XYZW(4), fov_h, fov_w]
    preds["depth"], ["depth_conf"]    # (1, S, H, W, 1), (1, S, H, W) fp32
    preds["world_points"], [..._conf] # (1, S, H, W, 3), (1, S, H, W) fp32
    kept, psi = model.aggregator(images)  # {layer: (1, S, N, 2C) bf16}, patch_start_idx

Under torchrun with world_size > 1 (`dist=True`) the views are frame-sharded:
every rank passes the FULL image batch (or its own slice with `sharded_input`),
the global attention layers run the K/V ring (ring.py), the camera head sees
all camera tokens (all-gather), and the dense outputs returned are this rank's
frame slice while `pose_enc` is global.
"""
from __future__ import annotations

from typing import Dict, Optional, Tuple

import torch

from . import ops
from .aggregator import DeviceWeights, aggregator_forward, alloc_workspace
from .config import VGGTConfig, vggt_1b
from .heads import DPTHeadDevice, camera_head
from .profiling import phase
from .pose import pose_encoding_to_extri_intri  # noqa: F401  (re-export, upstream location)
from .weights import check_state_dict, make_state_dict


def _require_b200(device):
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_25191_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    cap = torch.cuda.get_device_capability(device)
    if cap[0] != 10:
        raise RuntimeError(f"sm_100a kernels need a Blackwell B200 (got compute capability {cap})")


class VGGT:
    def __init__(self, cfg: Optional[VGGTConfig] = None, state_dict=None, seed: int = 0, device="cuda",
                 dist: bool = False, comm=None):
        """dist=True: frame-sharded over the ranks of torch.distributed (or of `comm`, an object with
        rank / world / sendrecv / all_gather like ring.TorchDistComm)."""
        self.cfg = cfg or vggt_1b()
        self.device = torch.device(device)
        _require_b200(self.device)
        ops.load_library()
        sd = state_dict if state_dict is not None else make_state_dict(self.cfg, seed)
        check_state_dict(sd, self.cfg)
        self.W = DeviceWeights(sd, self.cfg, self.device)
        self.depth_head = DPTHeadDevice(self.W, "depth_head.", "exp")
        self.point_head = DPTHeadDevice(self.W, "point_head.", "inv_log")
        self.dist = dist
        self._streams = None
        self.ring = None
        if dist:
            from .ring import FrameShardedRing
            self.ring = FrameShardedRing(self.cfg, self.device, comm=comm, q_log2=True)

    # -- helpers ------------------------------------------------------------
    def _head_streams(self, dev):
        if self._streams is None:
            self._streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        return self._streams

    def _local(self, images: torch.Tensor, sharded_input: bool):
        """(this rank's images on the device, global frame offset, global S).

        Host inputs are sliced to the rank's frames BEFORE the host-to-device copy, so every rank
        moves only its own views over PCIe."""
        if images.dim() == 5:
            if images.shape[0] != 1:
                raise ValueError("one scene per call here (forward / aggregator loop over B)")
            images = images[0]
        if images.dim() != 4 or images.shape[1] != 3:
            raise ValueError(f"images must be (S,3,H,W) or (1,S,3,H,W); got {tuple(images.shape)}")
        if self.ring is None:
            local, f0, S = images, 0, images.shape[0]
        else:
            local, f0, S = self.ring.local_frames(images, sharded_input)
        return local.to(self.device, torch.float32, non_blocking=True).contiguous(), f0, S

    # -- API ------------------------------------------------------------------
    @staticmethod
    def _scenes(images: torch.Tensor):
        """(B, S, 3, H, W) with B > 1: the upstream batch of independent scenes, run one after another."""
        return [images[b:b + 1] for b in range(images.shape[0])] if images.dim() == 5 and images.shape[0] > 1 else None

    @torch.no_grad()
    def aggregator(self, images: torch.Tensor, sharded_input: bool = False) -> Tuple[Dict[int, torch.Tensor], int]:
        scenes = self._scenes(images)
        if scenes is not None:
            parts = [self.aggregator(x, sharded_input)[0] for x in scenes]
            return {i: torch.cat([p[i] for p in parts]) for i in parts[0]}, self.cfg.patch_start_idx
        local, f0, S = self._local(images, sharded_input)
        kept = self._aggregate(local, f0)
        return {i: t[None] for i, t in kept.items()}, self.cfg.patch_start_idx

    def _aggregate(self, local: torch.Tensor, f0: int) -> Dict[int, torch.Tensor]:
        if self.ring is None:
            S, qc = local.shape[0], self.cfg.q_chunk
            ws = alloc_workspace(self.cfg, S, self.device, q_frames=qc if qc and S > qc else None)
            gattn = None
        else:  # K/V produced straight into the ring's send buffer, ring buffers allocated once per forward
            self.ring.begin()
            ws = alloc_workspace(self.cfg, local.shape[0], self.device, rows_per_head=self.ring.rows_per_head,
                                 kv=self.ring.kv_buffers())
            gattn = self.ring.global_attention
        kept = aggregator_forward(self.W, local, ws, global_attn=gattn, frame0_is_first=(f0 == 0))
        del ws
        return kept

    @torch.no_grad()
    def forward(self, images: torch.Tensor, sharded_input: bool = False) -> Dict[str, torch.Tensor]:
        scenes = self._scenes(images)
        if scenes is not None:  # outputs stacked along the upstream batch dimension B
            outs = [self.forward(x, sharded_input) for x in scenes]
            res = {k: torch.cat([o[k] for o in outs]) for k, v in outs[0].items() if isinstance(v, torch.Tensor)}
            res["pose_enc_list"] = [torch.cat([o["pose_enc_list"][i] for o in outs])
                                    for i in range(len(outs[0]["pose_enc_list"]))]
            res["frame_offset"] = outs[0]["frame_offset"]
            return res
        cfg = self.cfg
        local, f0, S = self._local(images, sharded_input)
        kept = self._aggregate(local, f0)
        Sl = local.shape[0]
        N = cfg.tokens_per_frame
        # camera head over ALL views (attention across camera tokens)
        cam = kept[cfg.kept_layers[-1]][:, 0]                      # (Sl, 2C) strided view
        if self.ring is not None:
            cam = self.ring.all_gather_frames(cam.contiguous())
        H = W = cfg.img_size
        dev = self.device
        depth = torch.empty(Sl, H, W, 1, device=dev)
        depth_conf = torch.empty(Sl, H, W, device=dev)
        pts = torch.empty(Sl, H, W, 3, device=dev)
        pts_conf = torch.empty(Sl, H, W, device=dev)
        # the three heads are independent: depth and point heads on two side streams, the camera head
        # concurrently on the current stream
        with phase("heads"):
            cur = torch.cuda.current_stream(dev)
            s_d, s_p = self._head_streams(dev)
            # the DPT heads' zero-bordered buffers come from the main stream's pool (allocated here, before
            # the side streams wait on it, and released after the main stream has waited for them), so the
            # next forward's aggregator reuses that memory
            F = min(Sl, cfg.head_chunk)
            self.depth_head.prepare(F, dev)
            self.point_head.prepare(F, dev)
            s_d.wait_stream(cur)
            s_p.wait_stream(cur)
            with torch.cuda.stream(s_d):
                self.depth_head(kept, depth, depth_conf, cfg.head_chunk)
            with torch.cuda.stream(s_p):
                self.point_head(kept, pts, pts_conf, cfg.head_chunk)
            pose_list = camera_head(self.W, cam)
            cur.wait_stream(s_d)
            cur.wait_stream(s_p)
            for t in kept.values():  # read on the side streams
                t.record_stream(s_d)
                t.record_stream(s_p)
            depth.record_stream(s_d)
            depth_conf.record_stream(s_d)
            pts.record_stream(s_p)
            pts_conf.record_stream(s_p)
            self.depth_head.release()  # freed into the main stream's pool, ordered after s_d / s_p above
            self.point_head.release()
        return {
            "pose_enc": pose_list[-1][None],
            "pose_enc_list": [p[None] for p in pose_list],
            "depth": depth[None],
            "depth_conf": depth_conf[None],
            "world_points": pts[None],
            "world_points_conf": pts_conf[None],
            "images": local[None],
            "frame_offset": f0,
        }

    __call__ = forward

    @torch.no_grad()
    def point_map_from_depth(self, preds: Dict[str, torch.Tensor]) -> torch.Tensor:
        """Depth-based world points (1, S_local, H, W, 3) fp32 from a forward's depth and decoded cameras
        (upstream `unproject_depth_map_to_point_map`; the point cloud VGGT-X uses to initialise 3DGS).
        Runs vx_unproject_depth; with frame sharding the cameras of this rank's frames are used."""
        from .scene import unproject_depth_maps
        depth = preds["depth"][0]
        S_local = depth.shape[0]
        f0 = int(preds.get("frame_offset", 0))
        enc = preds["pose_enc"][0, f0:f0 + S_local].float()
        extri, intri = pose_encoding_to_extri_intri(enc, tuple(depth.shape[1:3]))
        return unproject_depth_maps(depth, extri, intri)[None]
