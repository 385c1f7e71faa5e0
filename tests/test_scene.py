"""Scene-level consumers: matched points + depth sampling, dense depth
unprojection, view-angle pair selection and pose metrics.  The CPU oracle (oracle/scene_ref.py) is
pinned to the reference's own outputs (tests/golden/scene.npz from tests/golden/make_scene_golden.py);
the device implementation (paper_2509_25191_b200.scene / csrc/scene.cu) is checked against the same
goldens.  Integer / selection outputs (which correspondences survive, pair lists, flags, skip
counts) must match exactly; coordinates and angles to rounding (the reference's numpy / BLAS 3x3
products are not bit-reproducible), angles near 0 deg to the arccos conditioning.
"""
from pathlib import Path

import numpy as np
import pytest

from oracle import scene_ref

G = np.load(Path(__file__).parent / "golden" / "scene.npz")
MP = {k[3:]: G[k] for k in G.files if k.startswith("mp/")}


def _kinv(intr):
    return np.stack([scene_ref.k_inverse(*x[:4]) for x in intr])


CASES = [("sparse", 0.0), ("sparse", 0.3), ("sparse", 0.7), ("dense", 0.3)]


# ---------------------------------------------------------------------------------------------- CPU
def test_oracle_sample_depth_matches_reference():
    uv = G["sd/uv"]
    for key, dm in (("sd/sparse", MP["depth_sparse"][0]), ("sd/dense", MP["depth_dense"][1])):
        got = np.array([scene_ref.sample_depth(dm, u, v) for u, v in uv])
        np.testing.assert_array_equal(got, G[key])


@pytest.mark.parametrize("name,thr", CASES)
def test_oracle_matched_points_match_reference(name, thr):
    dm = MP[f"depth_{name}"]
    pts, sc, sk = scene_ref.select_matched_points(MP["pair_ij"], MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"],
                                                  {f: dm[f] for f in range(len(dm))}, MP["R"], MP["t"], MP["intr"],
                                                  thr)
    assert sk == int(G[f"mp/{name}_{thr}/skipped"])
    np.testing.assert_allclose(pts, G[f"mp/{name}_{thr}/points"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(sc, G[f"mp/{name}_{thr}/consistency"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("thr", [15.0, 30.0, 100.0, 180.0])
def test_oracle_select_pairs_matches_reference(thr):
    pairs, ang = scene_ref.select_pairs(G["sp/R"], thr)
    np.testing.assert_array_equal(pairs, G[f"sp/{thr}/pairs"])
    np.testing.assert_allclose(ang, G[f"sp/{thr}/angles"], rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("oi", [0, 1])
def test_oracle_pose_metrics_match_reference(oi):
    rre, rte, fl = scene_ref.pairwise_errors(G["pe/Rp"], G["pe/tp"], G["pe/Rg"], G["pe/tg"], G["pe/gt_of"], bool(oi))
    np.testing.assert_array_equal(fl, G[f"pe/{oi}/flags"])
    np.testing.assert_allclose(rre, G[f"pe/{oi}/rre"], rtol=1e-9, atol=1e-6)
    np.testing.assert_allclose(rte, G[f"pe/{oi}/rte"], rtol=1e-9, atol=1e-6)
    s = G[f"pe/{oi}/summary"]
    assert scene_ref.auc_at_30(rre, rte) == pytest.approx(s[3], rel=1e-9)


# ---------------------------------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def sc():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2509_25191_b200 import scene
    return scene


@pytest.mark.gpu
@pytest.mark.parametrize("name,thr", CASES)
@pytest.mark.parametrize("f32", [False, True])
def test_device_matched_points_match_reference(sc, name, thr, f32):
    import torch
    dm = MP[f"depth_{name}"]
    if f32:
        # fp32 maps (VGGT's output dtype) widen exactly: compare against the oracle on the same values
        dm32 = dm.astype(np.float32)
        maps = {f: torch.as_tensor(dm32[f]) for f in range(len(dm))}
        ref_pts, ref_sc, ref_sk = scene_ref.select_matched_points(
            MP["pair_ij"], MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"],
            {f: dm32[f].astype(np.float64) for f in range(len(dm))}, MP["R"], MP["t"], MP["intr"], thr)
    else:
        maps = {f: dm[f] for f in range(len(dm))}
        ref_pts, ref_sc, ref_sk = (G[f"mp/{name}_{thr}/points"], G[f"mp/{name}_{thr}/consistency"],
                                   int(G[f"mp/{name}_{thr}/skipped"]))
    pts, cons, sk = sc.select_matched_points_arrays(MP["pair_ij"], MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"],
                                                    maps, MP["R"], MP["t"], _kinv(MP["intr"]), thr)
    assert sk == ref_sk and pts.shape == ref_pts.shape
    np.testing.assert_allclose(pts, ref_pts, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(cons, ref_sc, rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
def test_device_matched_points_missing_map_and_threshold(sc):
    dm = MP["depth_sparse"]
    maps = {f: dm[f] for f in range(len(dm) - 1)}
    with pytest.raises(sc.MissingDepthMap):
        sc.select_matched_points_arrays(MP["pair_ij"], MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"], maps, MP["R"],
                                        MP["t"], _kinv(MP["intr"]), 0.3)
    with pytest.raises(ValueError):
        sc.select_matched_points_arrays(MP["pair_ij"], MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"], maps, MP["R"],
                                        MP["t"], _kinv(MP["intr"]), -0.1)


class _Obj:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _rig(R, t, ids=None):
    fr = tuple(_Obj(frame_id=(ids[k] if ids else f"f{k}"), pose=_Obj(R=R[k], t=t[k]),
                    intrinsics=_Obj(fx=400.0, fy=400.0, cx=319.5, cy=239.5)) for k in range(len(R)))
    return _Obj(frames=fr)


@pytest.mark.gpu
@pytest.mark.parametrize("thr", [15.0, 30.0, 100.0, 180.0])
def test_device_select_pairs_matches_reference(sc, thr):
    R = G["sp/R"]
    sel = sc.select_pairs(_rig(R, np.zeros((len(R), 3))), thr)
    np.testing.assert_array_equal(np.array(sel.pairs, dtype=np.int64).reshape(-1, 2), G[f"sp/{thr}/pairs"])
    np.testing.assert_allclose(sel.view_angle_deg, G[f"sp/{thr}/angles"], rtol=1e-12, atol=1e-9)
    with pytest.raises(ValueError):
        sc.select_pairs(_rig(R, np.zeros((len(R), 3))), 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("oi", [0, 1])
def test_device_pose_metrics_match_reference(sc, oi):
    n = len(G["pe/Rp"])
    ids_g = [f"g{k}" for k in range(n)]
    ids_p = [ids_g[g] for g in G["pe/gt_of"]]
    m = sc.evaluate_poses(_rig(G["pe/Rp"], G["pe/tp"], ids_p), _rig(G["pe/Rg"], G["pe/tg"], ids_g), bool(oi))
    np.testing.assert_array_equal(m.zero_baseline_flags, G[f"pe/{oi}/flags"])
    np.testing.assert_allclose(m.rre_deg, G[f"pe/{oi}/rre"], rtol=1e-9, atol=1e-6)
    np.testing.assert_allclose(m.rte_deg, G[f"pe/{oi}/rte"], rtol=1e-9, atol=1e-6)
    s = G[f"pe/{oi}/summary"]
    assert m.pair_count == int(s[2])
    assert m.rre_mean == pytest.approx(s[0], rel=1e-9, abs=1e-7)
    assert m.rte_mean == pytest.approx(s[1], rel=1e-9, abs=1e-7)
    assert m.auc_at_30 == pytest.approx(s[3], rel=1e-9)
    with pytest.raises(sc.FrameMismatch):
        sc.pairwise_errors(_rig(G["pe/Rp"], G["pe/tp"], ids_p), _rig(G["pe/Rg"][:3], G["pe/tg"][:3]))


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W", [(3, 37, 52), (2, 518, 518), (1, 7, 5)])
def test_device_unproject_depth_maps(sc, S, H, W):
    import torch
    g = torch.Generator().manual_seed(S * H)
    depth = 1 + torch.rand(S, H, W, generator=g)
    q = torch.nn.functional.normalize(torch.randn(S, 4, generator=g), dim=-1)
    from paper_2509_25191_b200.pose import quat_to_mat
    R = quat_to_mat(q)
    t = torch.randn(S, 3, 1, generator=g)
    extri = torch.cat([R, t], -1).float()
    intri = torch.tensor([[300.0, 0, W / 2], [0, 310.0, H / 2], [0, 0, 1]]).expand(S, 3, 3).contiguous()
    out = sc.unproject_depth_maps(depth.cuda(), extri.cuda(), intri.cuda()).cpu().double().numpy()
    ref = scene_ref.unproject_depth_maps(depth.double().numpy(), extri.double().numpy(), intri.double().numpy())
    scale = np.abs(ref).max()
    assert np.abs(out - ref).max() < 1e-5 * scale


@pytest.mark.gpu
def test_device_matched_points_mixed_map_sizes(sc):
    """Per-frame depth maps of different sizes and dtypes (DepthMap-like objects): the kernel's map
    table (offset, h, w per map) against the oracle."""
    rng = np.random.default_rng(4)
    dm = MP["depth_dense"]
    maps = {}
    for f in range(len(dm)):
        h, w = dm.shape[1] - 7 * (f % 3), dm.shape[2] - 5 * (f % 2)
        maps[f] = np.ascontiguousarray(dm[f, :h, :w])

    class _DM:
        def __init__(self, v):
            self.values = v

    objs = {f: _DM(v) for f, v in maps.items()}
    w = rng.uniform(0, 1, MP["w"].shape[0])
    ref_pts, ref_sc, ref_sk = scene_ref.select_matched_points(MP["pair_ij"], MP["offsets"], MP["xy_i"], MP["xy_j"], w,
                                                              maps, MP["R"], MP["t"], MP["intr"], 0.3)
    pts, cons, sk = sc.select_matched_points_arrays(MP["pair_ij"], MP["offsets"], MP["xy_i"], MP["xy_j"], w, objs,
                                                    MP["R"], MP["t"], _kinv(MP["intr"]), 0.3)
    assert sk == ref_sk and pts.shape == ref_pts.shape
    np.testing.assert_allclose(pts, ref_pts, rtol=1e-12, atol=1e-12)


def test_matched_points_rejects_out_of_rig_frame_index():
    """A pair naming a frame past the rig fails like the reference's rig[frame] (IndexError), before any
    device work (the kernel would otherwise read past the camera arrays)."""
    from paper_2509_25191_b200 import scene
    dm = MP["depth_sparse"]
    n = len(MP["R"])
    pij = MP["pair_ij"].copy()
    pij[0, 1] = n
    maps = {f: dm[0] for f in range(n + 1)}
    with pytest.raises(IndexError):
        scene.select_matched_points_arrays(pij, MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"], maps, MP["R"],
                                           MP["t"], _kinv(MP["intr"]), 0.3)
    pij[0, 1] = -n - 1
    maps[-n - 1] = dm[0]
    with pytest.raises(IndexError):
        scene.select_matched_points_arrays(pij, MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"], maps, MP["R"],
                                           MP["t"], _kinv(MP["intr"]), 0.3)


@pytest.mark.gpu
def test_device_matched_points_negative_frame_index_wraps(sc):
    """rig[-1] wraps in the reference while the depth map is looked up under the key -1."""
    dm = MP["depth_dense"]
    n = len(MP["R"])
    pij = MP["pair_ij"].copy()
    j_old = int(pij[0, 1])
    pij[0, 1] = j_old - n  # same camera, negative index
    depths = {f: dm[f] for f in range(len(dm))}
    depths[j_old - n] = dm[(j_old + 1) % len(dm)]  # a different map under the negative key
    ref_pts, ref_sc, ref_sk = scene_ref.select_matched_points(pij, MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"],
                                                              depths, MP["R"], MP["t"], MP["intr"], 0.3)
    pts, cons, sk = sc.select_matched_points_arrays(pij, MP["offsets"], MP["xy_i"], MP["xy_j"], MP["w"], depths,
                                                    MP["R"], MP["t"], _kinv(MP["intr"]), 0.3)
    assert sk == ref_sk and pts.shape == ref_pts.shape
    np.testing.assert_allclose(pts, ref_pts, rtol=1e-12, atol=1e-12)
