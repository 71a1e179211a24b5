"""GPU ground truth, occupancy and metrics (scene.cu) vs the restatements.

* render_gt on the GPU is bit-identical to synthetic.render_gt (the numpy
  restatement of generate_dataset's pixel loop, pinned against the reference)
  and to the reference built without FMA contraction where oracle/_ref exists.
* The GPU occupancy pipeline (ground truth -> back-projection -> device octree
  build) gives the same octree as the host pipeline.
* psnr / depth_errors / ssim match the reference formulas (src/metrics.cpp)
  in fp64 to 1e-12 relative (ssim also against the reference itself where
  oracle/_ref exists).
"""
import numpy as np
import pytest
import torch

import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = P.Context(0)
    yield c
    c.close()


def _ref_nofma():
    from oracle import Reference, reference_available

    return Reference(nofma=True) if reference_available(nofma=True) else None


@pytest.mark.parametrize("objects", [4, 20])
def test_render_gt_bit_exact(ctx, objects):
    reference_nofma = _ref_nofma()
    sc = S.make_random_scene(7, objects)
    cams = S.hemisphere_cameras(3, 1.8, 7, 96, 64, 100.0)
    for cam in cams:
        got = S.render_gt_gpu(ctx, sc, cam, 96, 64)
        want = S.render_gt(sc, cam, 96, 64)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
        if reference_nofma is not None:
            rs = reference_nofma.scene_make(7, objects)
            ref = reference_nofma.scene_render_gt(rs, cam, 96, 64)
            for a, b in zip(got, ref):
                assert np.array_equal(a, b)


def test_gpu_occupancy_pipeline(ctx):
    sc = S.make_random_scene(7, 4)
    cams = S.hemisphere_cameras(12, 1.8, 7, 160, 160, 240.0)
    g = P.GridConfig(128, dilation=1)
    tree, n = S.occupancy_octree_gpu(ctx, sc, cams, 160, 160, g)
    pts = S.occupancy_points(sc, cams, 160, 160)
    assert n == pts.shape[0]
    host = P.SparseOctree.build(pts, g, None)
    assert tree.vertex_count == host.vertex_count and tree.dropped_points == host.dropped_points
    for l in range(host.leaf_level + 1):
        assert np.array_equal(tree.level_codes(l), host.level_codes(l))
    assert np.array_equal(tree.corner_ids(), host.corner_ids())


def test_metrics(ctx):
    rng = np.random.default_rng(5)
    gt = rng.random(3 * 5000).astype(np.float32)
    pred = np.clip(gt + rng.normal(0, 0.02, gt.shape), 0, 1).astype(np.float32)
    d = lambda a: torch.from_numpy(a).cuda()
    tp, tg = d(pred), d(gt)
    torch.cuda.synchronize()
    got = P.psnr_device(ctx, tp.data_ptr(), tg.data_ptr(), gt.size)
    mse = np.mean((pred.astype(np.float64) - gt.astype(np.float64)) ** 2)
    assert got == pytest.approx(10 * np.log10(1 / mse), rel=1e-12)
    assert P.psnr_device(ctx, tg.data_ptr(), tg.data_ptr(), gt.size) == 99.0
    gd = rng.random(5000).astype(np.float32)
    pd = (gd + rng.normal(0, 0.01, gd.shape)).astype(np.float32)
    gm = (rng.random(5000) > 0.3).astype(np.float32)
    a, b, c = d(pd), d(gd), d(gm)
    torch.cuda.synchronize()
    rmse, mae, empty = P.depth_errors_device(ctx, a.data_ptr(), b.data_ptr(), c.data_ptr(), 5000)
    e = (pd.astype(np.float64) - gd)[gm >= 0.5]
    assert not empty
    assert rmse == pytest.approx(np.sqrt(np.mean(e * e)), rel=1e-12)
    assert mae == pytest.approx(np.mean(np.abs(e)), rel=1e-12)
    z = d(np.zeros(5000, np.float32))
    torch.cuda.synchronize()
    assert P.depth_errors_device(ctx, a.data_ptr(), b.data_ptr(), z.data_ptr(), 5000) == (0.0, 0.0, True)


@pytest.mark.parametrize("w,h,c", [(96, 64, 3), (11, 11, 1), (1600, 40, 3)])
def test_ssim_device(ctx, w, h, c):
    from oracle import Reference, reference_available, ssim

    rng = np.random.default_rng(w + h + c)
    gt = rng.random(w * h * c).astype(np.float32)
    pred = np.clip(gt + rng.normal(0, 0.03, gt.shape), 0, 1).astype(np.float32)
    tp, tg = torch.from_numpy(pred).cuda(), torch.from_numpy(gt).cuda()
    torch.cuda.synchronize()
    got = P.ssim_device(ctx, tp.data_ptr(), tg.data_ptr(), w, h, c)
    assert got == pytest.approx(ssim(pred, gt, w, h, c), rel=1e-12)
    if reference_available():
        assert got == pytest.approx(Reference().metrics(pred, gt, w, h, c)[1], rel=1e-12)
    assert P.ssim_device(ctx, tg.data_ptr(), tg.data_ptr(), w, h, c) == pytest.approx(1.0, rel=1e-14)
    with pytest.raises(ValueError, match="SSIM window"):
        P.ssim_device(ctx, tp.data_ptr(), tg.data_ptr(), 10, h, c)
