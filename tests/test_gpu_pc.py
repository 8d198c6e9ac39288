"""Point-cloud brute force on the GPU vs the reference: masks bit-exact, FIMs <= 1e-4 relative."""
import numpy as np
import pytest
import torch

import paper_2008_03324_b200 as F

pytestmark = pytest.mark.gpu


def relf(a, b):
    a, b = a.reshape(len(a), -1), b.reshape(len(b), -1)
    return np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-300)


def test_pc_vs_reference_golden(g_pc):
    cam = F.PinholeCamera.from_fov()
    out = F.exact_pose_fim_batch(g_pc["rotations"], g_pc["translations"], g_pc["points"], cam)
    assert relf(out, g_pc["fims"]).max() <= 1e-5
    dev = torch.device("cuda")
    mask = torch.zeros((g_pc["rotations"].shape[0], g_pc["points"].shape[0]), dtype=torch.uint8, device=dev)
    F.exact_pose_fim_batch_device(torch.tensor(g_pc["rotations"].reshape(-1, 9), device=dev),
                                  torch.tensor(g_pc["translations"], device=dev),
                                  torch.tensor(g_pc["points"], device=dev), cam, mask=mask)
    assert np.array_equal(mask.cpu().numpy().astype(bool), g_pc["visible_kernel"])


def test_pc_config3_sample_vs_oracle(oracle):
    from paper_2008_03324_b200 import scenes

    w = scenes.config3(3000)
    cam = F.PinholeCamera.from_fov()
    dev = torch.device("cuda")
    r = torch.tensor(w.rotations.reshape(-1, 9), device=dev)
    t = torch.tensor(w.positions, device=dev)
    p = torch.tensor(w.points, device=dev)
    mask = torch.zeros((3000, w.points.shape[0]), dtype=torch.uint8, device=dev)
    out = F.exact_pose_fim_batch_device(r, t, p, cam, mask=mask).cpu().numpy().reshape(-1, 6, 6)
    ref = oracle.exact_fim_batch(w.rotations, w.positions, w.points, cam.as_tuple())
    om = oracle.pc_mask(w.rotations, w.positions, w.points, cam.as_tuple())
    assert np.array_equal(mask.cpu().numpy().astype(bool), om)  # 6e7 pairs, bit-exact
    assert relf(out, ref).max() <= 1e-4


def test_pc_border_and_edge_cases(oracle):
    cam = F.PinholeCamera.from_fov()
    rng = np.random.default_rng(8)
    R = np.stack([F.random_rotation(rng) for _ in range(8)])
    t = rng.uniform(-1, 1, size=(8, 3))
    pts = []
    for q in range(8):  # landmarks on the exact pixel borders u,v in {0, 640} at several depths
        for zc in (0.7, 1.0, 3.3):
            for u, v in ((0.0, 50.0), (640.0, 70.0), (90.0, 0.0), (100.0, 640.0), (320.0, 320.0)):
                pc = np.array([(u - cam.cx) * zc / cam.fx, (v - cam.cy) * zc / cam.fy, zc])
                pts.append(R[q] @ pc + t[q])
    pts.append(t[0])  # on a camera centre: zc = 0 -> invisible
    pts = np.array(pts)
    out = F.exact_pose_fim_batch(R, t, pts, cam)
    ref = oracle.exact_fim_batch(R, t, pts, cam.as_tuple())
    assert relf(out, ref).max() <= 1e-4
    dev = torch.device("cuda")
    mask = torch.zeros((8, len(pts)), dtype=torch.uint8, device=dev)
    F.exact_pose_fim_batch_device(torch.tensor(R.reshape(-1, 9), device=dev), torch.tensor(t, device=dev),
                                  torch.tensor(pts, device=dev), cam, mask=mask)
    assert np.array_equal(mask.cpu().numpy().astype(bool), oracle.pc_mask(R, t, pts, cam.as_tuple()))
    # empty scene -> zeros (fim.py:141-142)
    assert np.all(F.exact_pose_fim_batch(R, t, np.zeros((0, 3)), cam) == 0)
    single = F.exact_pose_fim(F.Pose(R[0], t[0]), pts, cam)
    assert np.allclose(single, out[0], rtol=1e-12, atol=0)


def test_pc_pose_order_is_invisible():
    """Large batches run similar poses together (load balance); per-pose results and masks
    are bit-identical to batches below the reordering threshold."""
    from paper_2008_03324_b200 import scenes

    w = scenes.config3(12000)
    cam = F.PinholeCamera.from_fov()
    dev = torch.device("cuda")
    r = torch.tensor(w.rotations.reshape(-1, 9), device=dev)
    t = torch.tensor(w.positions, device=dev)
    p = torch.tensor(w.points[:5000], device=dev)
    m_all = torch.zeros((12000, 5000), dtype=torch.uint8, device=dev)
    o_all = F.exact_pose_fim_batch_device(r, t, p, cam, mask=m_all)
    for s in range(0, 12000, 4000):
        m = torch.zeros((4000, 5000), dtype=torch.uint8, device=dev)
        o = F.exact_pose_fim_batch_device(r[s:s + 4000].contiguous(), t[s:s + 4000].contiguous(), p, cam, mask=m)
        assert torch.equal(o, o_all[s:s + 4000])
        assert torch.equal(m, m_all[s:s + 4000])
