"""The maintainer-side ctypes binding shown in INTEGRATION.md, executed as written: its
build_quad_factors / build_gp_factors / exact_fim_batch / match_mask must reproduce the
reference (golden fixtures and the pinned C oracle) through the C ABI."""
import os
import re

import numpy as np
import pytest

import paper_2008_03324_b200 as F

from ._helpers import info_rel_fro

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def stub():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = next(b for b in re.findall(r"```python\n(.*?)```", text, re.S) if "kernels_cuda.py" in b)
    ns: dict = {}
    exec(compile(block, "INTEGRATION.md:kernels_cuda", "exec"), ns)
    return ns


def _scene(seed=3, n=300):
    rng = np.random.default_rng(seed)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(n, 3))
    grid = F.GridConfig(np.array([-2.0, -2.0, 0.0]), 0.5, np.array([8, 8, 4]))
    return pts, grid.centers()


def test_stub_quad_build_bit_identical(stub, oracle):
    pts, cen = _scene()
    q = F.build_quad_model()
    for trace in (True, False):
        mine = stub["build_quad_factors"](cen, pts, 1.0, q.k2, q.k1, q.k0, trace)
        ref = oracle.build_quad_factors(cen, pts, 1.0, q.k2, q.k1, q.k0, trace)
        assert np.array_equal(mine, ref)


def test_stub_gp_build(stub, oracle):
    pts, cen = _scene()
    m = F.build_gp_model(30)
    for trace in (True, False):
        mine = stub["build_gp_factors"](cen, pts, 1.0, m.samples, m.kinv, m.k_s, np.cos(m.alpha), trace,
                                        m.params.sigma2, m.params.length_scale)
        ref = oracle.build_gp_factors(cen, pts, 1.0, m.samples, m.kinv, m.k_s, np.cos(m.alpha), trace)
        assert info_rel_fro(mine, ref).max() <= 1e-4


def test_stub_pc_and_mask(stub, oracle, g_pc):
    cam = F.PinholeCamera.from_fov()
    out = stub["exact_fim_batch"](g_pc["rotations"], g_pc["translations"], g_pc["points"], *cam.as_tuple(), 1.0)
    ref = g_pc["fims"]
    rel = np.linalg.norm((out - ref).reshape(len(ref), -1), axis=1) / np.maximum(
        np.linalg.norm(ref.reshape(len(ref), -1), axis=1), 1e-300)
    assert rel.max() <= 1e-5
    pts, cen = _scene(5, 200)
    vd = np.random.default_rng(5).normal(size=(200, 3))
    vd /= np.linalg.norm(vd, axis=1, keepdims=True)
    mine = stub["match_mask"](cen, pts, vd, d_near=0.3, d_far=3.0, beta=np.pi / 3)
    want = F.Matchability(d_near=0.3, d_far=3.0, view_cone_beta=np.pi / 3).mask(cen, pts, vd)
    assert np.array_equal(mine.astype(bool), np.asarray(want, dtype=bool))
