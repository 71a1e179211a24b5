"""The C restatement against the UNMODIFIED reference compiled here
(oracle/_ref). Skipped where oracle/_ref is absent. Bit-exact against the
-ffp-contract=off build: octree, camera rays, hit lists (ids, order, t),
init_model, render_frame, Adam; losses and feature gradients identical,
decoder weight gradients relative L2 < 1e-6 (the reference reduces them in
omp-simd order)."""
import numpy as np
import pytest

import paper_2205_07058_b200.synthetic as S


@pytest.fixture(scope="module")
def c1(oracle, reference_nofma):
    pts, res, dil, cam, W, H = S.c1_workload()
    return pts, res, dil, cam, W, H, oracle.tree_build(pts, res, dil), reference_nofma.tree_build(pts, res, dil)


def test_octree_and_camera(c1, oracle, reference_nofma):
    pts, res, dil, cam, W, H, to, tr = c1
    for l in range(to.leaf_level + 1):
        assert np.array_equal(to.level_codes(l), tr.level_codes(l))
    assert np.array_equal(to.corner_ids, tr.corner_ids) and to.vertex_count == tr.vertex_count
    eye = tuple(0.5 + 1.8 * c for c in S.C1_EYE_DIR)
    assert np.array_equal(oracle.lookat_camera(eye, (0.5, 0.5, 0.5), W, H, 300.0),
                          reference_nofma.lookat_camera(eye, (0.5, 0.5, 0.5), W, H, 300.0))
    assert np.array_equal(oracle.camera_rays(cam, W, H), reference_nofma.camera_rays(cam, W, H))


def test_traversal_c1(c1, oracle, reference_nofma, reference):
    pts, res, dil, cam, W, H, to, tr = c1
    rays = oracle.camera_rays(cam, W, H)
    a = oracle.traverse(to, rays)
    b = reference_nofma.traverse(tr, rays)
    c = reference.traverse(reference.tree_build(pts, res, dil), rays)
    assert a[1].size == 59905
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.array_equal(a[0], c[0]) and np.array_equal(a[1], c[1])  # ids/order also vs the FMA build


def test_render_c1(c1, oracle, reference_nofma):
    pts, res, dil, cam, W, H, to, tr = c1
    m = oracle.init_model(to, 1)
    mr = reference_nofma.init_model(tr, 1)
    for k in ("ft", "fc", "mt", "mc"):
        assert np.array_equal(getattr(m, k), getattr(mr, k))
    a = oracle.render_frame(to, m, cam, W, H)
    b = reference_nofma.render_frame(tr, m, cam, W, H)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_scene_generator_matches_reference(oracle, reference_nofma):
    cams = oracle.hemisphere_cameras(3, 1.8, 7, 40, 40, 60.0)
    assert np.array_equal(cams, reference_nofma.hemisphere_cameras(3, 1.8, 7, 40, 40, 60.0))
    for prims in (4, 20):
        so, sr = oracle.scene_make(7, prims), reference_nofma.scene_make(7, prims)
        for c in cams:
            for x, y in zip(oracle.scene_render_gt(so, c, 40, 40), reference_nofma.scene_render_gt(sr, c, 40, 40)):
                assert np.array_equal(x, y)


@pytest.mark.parametrize("mode,frozen,lw", [(0, False, (1.0, 0.01, 0.01, 0.1)), (0, False, (1.0, 0.01, 0.0, 0.1)),
                                            (1, False, (1.0, 0.01, 0.01, 0.1)), (1, True, (1.0, 0.01, 0.01, 0.1))])
def test_losses(oracle, reference_nofma, mode, frozen, lw):
    W = 32
    sc = S.make_random_scene(7, 4)
    cams = S.hemisphere_cameras(2, 1.8, 7, W, W, 1.5 * W)
    pts = S.occupancy_points(sc, cams, W, W)
    to, tr = oracle.tree_build(pts, 32, 1), reference_nofma.tree_build(pts, 32, 1)
    rgb, depth, mask = S.render_gt(sc, cams[0], W, W)
    rays = S.camera_rays(cams[0], W, W)
    m = oracle.init_model(to, 0)
    la, ga, sa = oracle.loss(to, m, rays, rgb, depth.astype(np.float64), mask > 0.5, mode, lw=lw, frozen=frozen)
    lb, gb, sb = reference_nofma.loss(tr, m, rays, rgb, depth.astype(np.float64), mask > 0.5, mode, lw=lw,
                                      frozen=frozen)
    assert la == lb and sa.tolist() == sb.tolist()
    assert np.array_equal(ga.ft, gb.ft) and np.array_equal(ga.fc, gb.fc)
    for k in ("mt", "mc"):
        x, y = getattr(ga, k), getattr(gb, k)
        nb = np.linalg.norm(y)
        assert (np.linalg.norm(x - y) / nb if nb else np.linalg.norm(x)) < 1e-6


def test_adam(oracle, reference_nofma):
    rng = np.random.default_rng(1)
    p = rng.standard_normal(500).astype(np.float32)
    g = (rng.standard_normal(500) * 1e-2).astype(np.float32)
    out = []
    for lib in (oracle, reference_nofma):
        pp, m, v = p.copy(), np.zeros(500, np.float32), np.zeros(500, np.float32)
        for step in range(3):
            lib.adam_step(pp, g, m, v, step, np.float32(2e-4))
        out.append((pp, m, v))
    for x, y in zip(*out):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("w,h,c", [(40, 30, 3), (11, 11, 1), (64, 17, 3)])
def test_metrics_port(reference, w, h, c):
    """oracle.ssim (numpy restatement of src/metrics.cpp:70-113) against the reference's ssim."""
    from oracle import ssim

    rng = np.random.default_rng(w * h + c)
    gt = rng.random(w * h * c).astype(np.float32)
    pred = np.clip(gt + rng.normal(0, 0.05, gt.shape), 0, 1).astype(np.float32)
    _, want = reference.metrics(pred, gt, w, h, c)
    assert ssim(pred, gt, w, h, c) == pytest.approx(want, rel=1e-13)
    assert reference.metrics(gt, gt, w, h, c) == (99.0, pytest.approx(1.0, rel=1e-15))
