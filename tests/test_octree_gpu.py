"""GPU octree build (octree_build.cu) vs the host build (host_octree.cpp, pinned
byte-identical to the reference by test_golden / test_oracle_vs_ref): every
level's codes, the corner vertex ids, vertex and dropped-point counts must be
identical, including points on the max faces, outside the box, dilation
clipping at the grid border and a non-unit scene box."""
import numpy as np
import pytest

import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = P.Context(0)
    yield c
    c.close()


def _same(a, b):
    assert a.leaf_level == b.leaf_level
    assert a.vertex_count == b.vertex_count
    assert a.dropped_points == b.dropped_points
    for l in range(a.leaf_level + 1):
        assert np.array_equal(a.level_codes(l), b.level_codes(l)), l
    assert np.array_equal(a.corner_ids(), b.corner_ids())


def _edge_points(rng, n):
    p = rng.random((n, 3))
    p[: n // 10] = rng.integers(0, 2, (n // 10, 3))          # corners / max faces exactly
    p[n // 10: n // 5] = rng.random((n // 10, 3)) * 1.4 - 0.2  # some outside
    return p


@pytest.mark.parametrize("res,dil", [(2, 0), (4, 1), (16, 0), (16, 3), (64, 1), (256, 1), (1024, 0)])
def test_gpu_build_matches_host(ctx, res, dil):
    rng = np.random.default_rng(res * 10 + dil)
    pts = _edge_points(rng, 20000)
    g = P.GridConfig(res, dilation=dil)
    _same(P.SparseOctree.build(pts, g, ctx), P.SparseOctree.build(pts, g, None))


def test_gpu_build_c2_occupancy_and_device_points(ctx):
    import torch

    pts = S.occupancy_points(S.make_random_scene(7, 4), S.hemisphere_cameras(20, 1.8, 7, 200, 200, 300.0), 200, 200)
    g = P.GridConfig(256, dilation=1)
    host = P.SparseOctree.build(pts, g, None)
    _same(P.SparseOctree.build(pts, g, ctx), host)
    d = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float64)).cuda()
    torch.cuda.synchronize()
    _same(P.SparseOctree.build_device(d.data_ptr(), pts.shape[0], g, ctx), host)


def test_gpu_build_box_and_errors(ctx):
    rng = np.random.default_rng(3)
    pts = rng.random((5000, 3)) * 4.0 - 1.0
    g = P.GridConfig(32, dilation=2, lo=(-1.0, -1.0, -1.0), hi=(3.0, 3.0, 3.0))
    _same(P.SparseOctree.build(pts, g, ctx), P.SparseOctree.build(pts, g, None))
    with pytest.raises(RuntimeError, match="empty occupancy"):
        P.SparseOctree.build(np.full((10, 3), 5.0), P.GridConfig(8), ctx)
    with pytest.raises(ValueError):
        P.SparseOctree.build(pts, P.GridConfig(12), ctx)
