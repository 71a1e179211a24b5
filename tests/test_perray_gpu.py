"""The reference's per-ray public API through the C ABI's batched GPU entries
(render.hpp:28-76, train.hpp:41, features.hpp:67-80): render_ray,
evaluate_voxel, composite, parameterize_ray, eta_gt, local_coords,
interpolate(_backward). Gates: bit-exact against the C restatement of the
reference (pinned to the no-FMA reference build) wherever the reference's
arithmetic is reproduced operand by operand; the reference's error messages.
"""
import numpy as np
import pytest

import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S

pytestmark = pytest.mark.gpu

HALF_SQRT3 = 0.5 * 1.7320508075688772


@pytest.fixture(scope="module")
def ctx():
    c = P.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def c1(ctx, oracle):
    pts, res, dil, cam, W, H = S.c1_workload()
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    otree = oracle.tree_build(pts, res, dil)
    model = P.Model(tree, seed=3, ctx=ctx)
    om = oracle.init_model(otree, 3)
    rays = oracle.camera_rays(cam, W, H)
    return tree, otree, model, om, rays


def test_render_ray_equals_the_frame_renderer(c1, oracle):
    """render_ray (single-ray path: traverse -> evaluate_voxel per hit -> composite -> expected
    depth) equals the reference's frame output for the same rays (the reference's render_ray
    equals render_frame exactly)."""
    tree, otree, model, om, rays = c1
    idx = np.flatnonzero(np.diff(tree.traverse(rays)[0]) > 0)[::40][:200]  # foreground rays
    orgb, oa, od, _ = oracle.render_rays(otree, om, rays[idx])
    for k, i in enumerate(idx):
        r = P.render_ray(model, rays[i])
        assert np.array_equal(np.float32(r["color"]), orgb[3 * k:3 * k + 3])
        assert np.float32(r["alpha"]) == oa[k]
        assert np.float32(r["expected_depth"]) == od[k]
        assert len(r["samples"]["tau"]) == len(r["samples"]["voxel_ids"]) > 0
    # a background ray: no samples, black, zero depth
    away = np.array([[0.5, 0.5, 3.0, 0.0, 0.0, 1.0]])
    r = P.render_ray(model, away)
    assert r["samples"]["voxel_ids"].size == 0 and r["alpha"] == 0.0 and r["expected_depth"] == 0.0


def test_evaluate_voxel_samples(c1):
    tree, otree, model, om, rays = c1
    off, ids, tin, tout = tree.traverse(rays[:4000])
    ray_of = np.repeat(np.arange(4000), np.diff(off))
    ev = P.evaluate_voxels(model, rays[:4000][ray_of], ids, tin, tout)
    assert ev["tau"].size == ids.size and np.all(ev["tau"] >= 0)
    assert np.all((ev["eta"] > 0) & (ev["eta"] < 1)) and np.all((ev["color"] >= 0) & (ev["color"] <= 1))
    # x_s = x1 eta + x2 (1 - eta) with eta the decoder's float (render.cpp:49), and t_s likewise
    r = rays[:4000][ray_of]
    x1, x2 = r[:, :3] + r[:, 3:] * tin[:, None], r[:, :3] + r[:, 3:] * tout[:, None]
    e = ev["eta"][:, None]
    assert np.array_equal(ev["x_s"], x1 * e + x2 * (1.0 - e))
    assert np.array_equal(ev["t_s"], ev["eta"] * tin + (1.0 - ev["eta"]) * tout)
    with pytest.raises(IndexError, match="unknown voxel id"):
        P.evaluate_voxels(model, rays[:1], np.array([12345678901], np.uint64), tin[:1], tout[:1])


def test_composite_matches_the_reference_recurrence(ctx):
    rng = np.random.default_rng(5)
    taus = rng.exponential(0.7, 37)
    cols = rng.uniform(0, 1, (37, 3))
    col, a, w, d = P.composite(taus, cols, t_s=np.linspace(1, 2, 37), ctx=ctx)
    T, c, al, ws = 1.0, np.zeros(3), 0.0, []
    for t, cc in zip(taus, cols):  # src/render.cpp:65-87 in double
        e = np.exp(-t)
        wi = T * (1.0 - e)
        c = c + wi * cc
        al += wi
        T *= e
        ws.append(wi)
    np.testing.assert_allclose(col[0], c, rtol=1e-15, atol=1e-16)
    # CUDA's and numpy's exp may differ by an ulp; the transmittance product carries it along
    assert abs(a[0] - al) <= 1e-14 and np.allclose(w, ws, rtol=0, atol=1e-14)
    assert abs(d[0] - np.dot(ws, np.linspace(1, 2, 37)) / al) <= 1e-14
    # several lists at once; an empty list composites to zero
    col2, a2, _, _ = P.composite(np.r_[taus, taus[:3]], np.r_[cols, cols[:3]], offsets=[0, 37, 37, 40], ctx=ctx)
    assert np.array_equal(col2[0], col[0]) and a2[1] == 0.0 and np.all(col2[1] == 0)
    with pytest.raises(ValueError, match="negative optical thickness"):
        P.composite([0.5, -1e-3], [[0, 0, 0], [1, 1, 1]], ctx=ctx)


def _parameterize_np(r, lo, hi):
    c = (lo + hi) * 0.5
    oc = r[:3] - c
    rad = HALF_SQRT3 * (hi[0] - lo[0])
    b = (oc[0] * r[3] + oc[1] * r[4]) + oc[2] * r[5]
    cc = ((oc[0] * oc[0] + oc[1] * oc[1]) + oc[2] * oc[2]) - rad * rad
    disc = b * b - cc
    s = np.sqrt(disc)
    p1 = r[:3] + r[3:] * (-b - s) - c
    p2 = r[:3] + r[3:] * (-b + s) - c
    n1 = np.sqrt((p1[0] * p1[0] + p1[1] * p1[1]) + p1[2] * p1[2])
    n2 = np.sqrt((p2[0] * p2[0] + p2[1] * p2[1]) + p2[2] * p2[2])
    return np.r_[p1 / n1, p2 / n2]


def test_parameterize_ray_bit_exact_and_tangent(c1, ctx):
    tree, otree, model, om, rays = c1
    off, ids, tin, tout = tree.traverse(rays[:3000])
    ray_of = np.repeat(np.arange(3000), np.diff(off))
    h = 1.0 / 64
    xyz = np.stack([np.array([sum(((int(c) >> (3 * b + a)) & 1) << b for b in range(21)) for a in range(3)])
                    for c in ids[:300]])
    boxes = np.c_[xyz * h, (xyz + 1) * h]
    got = P.parameterize_rays(rays[:3000][ray_of][:300], boxes, ctx=ctx)
    want = np.stack([_parameterize_np(rays[:3000][ray_of][k], boxes[k, :3], boxes[k, 3:]) for k in range(300)])
    assert np.array_equal(got, want)
    assert np.allclose(np.linalg.norm(got[:, :3], axis=1), 1.0) and np.allclose(np.linalg.norm(got[:, 3:], axis=1), 1.0)
    with pytest.raises(RuntimeError, match="tangent ray"):  # a ray passing far from the box's sphere
        P.parameterize_rays([[5.0, 5.0, 5.0, 1.0, 0.0, 0.0]], [[0, 0, 0, 0.1, 0.1, 0.1]], ctx=ctx)


def test_eta_gt(ctx):
    tin, tout = np.array([1.0, 1.0, 1.0, 2.0]), np.array([2.0, 2.0, 2.0, 2.5])
    d = np.array([1.25, 1.0 - 5e-7, 2.0 + 5e-7, 2.5])
    got = P.eta_gt(tin, tout, d, ctx=ctx)
    assert np.array_equal(got, np.clip((tout - d) / (tout - tin), 0.0, 1.0))
    with pytest.raises(RuntimeError, match="surface point outside voxel"):
        P.eta_gt([1.0], [2.0], [2.0 + 2e-6], ctx=ctx)


def test_interpolate_batch_and_backward(c1, ctx):
    """Batched interpolate / interpolate_backward on the model's own tree against a numpy restatement
    of src/features.cpp:33-84 (float accumulation in corner order; weights in double)."""
    tree, otree, model, om, rays = c1
    rng = np.random.default_rng(2)
    codes = tree.leaf_codes
    pick = codes[rng.integers(0, codes.size, 64)]
    h = 1.0 / 64
    lo = np.stack([np.array([sum(((int(c) >> (3 * b + a)) & 1) << b for b in range(21)) for a in range(3)])
                   for c in pick]) * h
    u = rng.uniform(0, 1, (64, 3))
    pts = lo + u * h
    vol = rng.uniform(-1, 1, (tree.vertex_count, 5)).astype(np.float32)
    got = P.interpolate(vol, tree, pick, pts, ctx=ctx)
    uu = P.local_coords(tree, pick, pts, ctx=ctx)
    assert np.array_equal(uu, np.clip((pts - lo) / h, 0, 1))
    corners = tree.corner_ids().reshape(-1, 8)
    index = {int(c): i for i, c in enumerate(codes)}
    want = np.zeros_like(got)
    for k in range(64):
        cs = corners[index[int(pick[k])]]
        for b in range(8):
            wx = uu[k, 0] if b & 1 else 1 - uu[k, 0]
            wy = uu[k, 1] if b & 2 else 1 - uu[k, 1]
            wz = uu[k, 2] if b & 4 else 1 - uu[k, 2]
            want[k] = want[k] + np.float32(wx * wy * wz) * vol[cs[b]]
    assert np.array_equal(got, want)
    grad = np.zeros_like(vol)
    P.interpolate_backward(vol, tree, pick[:1], pts[:1], np.ones((1, 5), np.float32), grad, ctx=ctx)
    cs = corners[index[int(pick[0])]]
    assert np.allclose(grad[cs].sum(axis=0), 1.0, atol=1e-6) and np.count_nonzero(grad.sum(axis=1)) <= 8
    with pytest.raises(RuntimeError, match="point not in voxel"):
        P.interpolate(vol, tree, pick[:1], pts[:1] + 2 * h, ctx=ctx)
