"""GPU parity: traversal and render through the C ABI vs the CPU oracle.

Bars (BASELINE.json north_star): voxel hit lists bit-exact (ids, order,
t_in, t_out, x1, x2); fp32 render max-abs <= 1e-3 on rgb/alpha/depth (the
kernel keeps the reference's accumulation order, so the observed error is
~1e-7); render statistics identical.
"""
import numpy as np
import pytest

import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S

pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-3  # north_star: RGB/depth max-abs <= 1e-3 with the fp32 MLP


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
    return tree, otree, cam, W, H


def _assert_hits_equal(got, want):
    off_g, ids_g, tin_g, tout_g = got[:4]
    off_w, ids_w, tin_w, tout_w = want[:4]
    assert np.array_equal(off_g, off_w)
    assert np.array_equal(ids_g, ids_w)
    assert np.array_equal(tin_g, tin_w)  # bit-exact doubles
    assert np.array_equal(tout_g, tout_w)


def test_traversal_c1_camera_rays_bit_exact(c1, oracle):
    tree, otree, cam, W, H = c1
    rays = oracle.camera_rays(cam, W, H)
    got = tree.traverse(rays, with_points=True)
    want = oracle.traverse(otree, rays)
    assert want[1].size == 59905  # C1 has 59,905 hits
    _assert_hits_equal(got, want)
    # x1/x2 = ray.at(t) exactly
    ray_of = np.repeat(np.arange(rays.shape[0]), np.diff(got[0]))
    o, d = rays[ray_of, :3], rays[ray_of, 3:]
    assert np.array_equal(got[4][:, :3], o + d * got[2][:, None])
    assert np.array_equal(got[4][:, 3:], o + d * got[3][:, None])


def test_traversal_node_tests_match_reference_walk(c1, ctx, oracle):
    """The traversal's ray-box test counter (bench's node-tests/s) equals the reference walk's ray_aabb calls
    (src/octree.cpp:185-235; 143.8 per C1 ray)."""
    tree, otree, cam, W, H = c1
    rays = oracle.camera_rays(cam, W, H)
    ctx.set_node_test_counting(True)
    try:
        tree.traverse(rays)
        got = ctx.last_node_tests()
    finally:
        ctx.set_node_test_counting(False)
    oracle.node_tests()
    oracle.traverse(otree, rays)
    want = oracle.node_tests() // 2  # oracle.traverse walks twice (count pass, then fill pass)
    assert got == want  # C1 has no re-traversed (overflowed) tiles, so no test is repeated
    assert abs(want / rays.shape[0] - 143.8) < 0.05


def test_traversal_reference_random_rays(ctx, oracle):
    """tests/test_octree.cpp:140-154: random 16^3 density-0.1 seed-7 octree, 1000 rays (Rng 11)."""
    pts = S.random_occupancy_points(16, 0.1, 7)
    tree = P.SparseOctree.build(pts, P.GridConfig(16, dilation=0), ctx)
    otree = oracle.tree_build(pts, 16, 0)
    rays = S.random_rays(11, 1000)
    _assert_hits_equal(tree.traverse(rays), oracle.traverse(otree, rays))


def test_traversal_tie_rule_grazing_face(ctx):
    """tests/test_octree.cpp:156-173: a ray in the shared x=0.5 face hits both leaves, Morton order."""
    pts = np.array([[0.25, 0.25, 0.25], [0.75, 0.25, 0.25]])
    tree = P.SparseOctree.build(pts, P.GridConfig(2, dilation=0), ctx)
    off, ids, tin, tout = tree.traverse(np.array([[0.5, -1.0, 0.25, 0.0, 1.0, 0.0]]))
    assert ids.size == 2 and ids[0] < ids[1] and tin[0] == tin[1]


def test_traversal_empty_and_missing_rays(ctx, oracle):
    pts = S.random_occupancy_points(16, 0.1, 7)
    tree = P.SparseOctree.build(pts, P.GridConfig(16, dilation=0), ctx)
    off, ids, *_ = tree.traverse(np.zeros((0, 6)))
    assert off.tolist() == [0] and ids.size == 0
    # rays pointing away from the cube
    rays = np.array([[2.0, 2.0, 2.0, 0.0, 0.0, 1.0], [-1.0, 0.5, 0.5, -1.0, 0.0, 0.0]])
    off, ids, *_ = tree.traverse(rays)
    assert off.tolist() == [0, 0, 0]


def test_traversal_many_hit_rays(ctx, oracle):
    """Long-tailed hit lists: a dense 64^3 block, diagonal rays."""
    pts = S.random_occupancy_points(64, 0.6, 3)
    tree = P.SparseOctree.build(pts, P.GridConfig(64, dilation=1), ctx)
    otree = oracle.tree_build(pts, 64, 1)
    rays = S.random_rays(5, 300)
    got, want = tree.traverse(rays), oracle.traverse(otree, rays)
    assert np.diff(want[0]).max() > 100
    _assert_hits_equal(got, want)
    # these rays overflow the first pass's queue: the partial hand-over (the rays reaching the
    # overflowing chunk leave the tile) and the second cooperative pass took part
    t = ctx.last_timings()
    assert t["dense_rays"] > 0 and t["hits"] == want[1].size


def test_render_c1_fp32(c1, oracle, ctx):
    tree, otree, cam, W, H = c1
    model = P.Model(tree, seed=1, ctx=ctx)
    om = oracle.init_model(otree, 1)
    ft, fc, mt, mc = model.get_params()
    assert np.array_equal(ft, om.ft) and np.array_equal(mt, om.mt) and np.array_equal(mc, om.mc)
    st = P.RenderStats()
    rgb, a, d = P.render_frame(model, P.Camera.from_record(cam, W, H), stats=st)
    orgb, oa, od, ost = oracle.render_frame(otree, om, cam, W, H)
    assert np.abs(rgb.reshape(-1) - orgb).max() <= TOL_FP32
    assert np.abs(a.reshape(-1) - oa).max() <= TOL_FP32
    assert np.abs(d.reshape(-1) - od).max() <= TOL_FP32
    assert [st.rays, st.rays_with_hits, st.traversal_hits, st.thickness_queries, st.color_queries] == list(ost)
    # the fp32 path keeps the reference's order: observed error is ulp-level
    assert np.abs(rgb.reshape(-1) - orgb).max() <= 1e-5


def test_render_background_and_rays_api(c1, oracle, ctx):
    tree, otree, cam, W, H = c1
    model = P.Model(tree, seed=3, ctx=ctx)
    om = oracle.init_model(otree, 3)
    rays = oracle.camera_rays(cam, W, H)[::7]
    bg = np.array([0.2, 0.5, 0.9], np.float32)
    rgb, a, d = P.render_rays(model, rays, background=bg)
    orgb, oa, od, _ = oracle.render_rays(otree, om, rays, bg=bg)
    assert np.abs(rgb.reshape(-1) - orgb).max() <= 1e-5
    assert np.abs(d - od).max() <= 1e-5


def test_render_rtmv_small_fp32(ctx, oracle):
    """RTMV-shaped scene (20 objects), reduced sizes so the oracle finishes in seconds."""
    sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=20, n_views=8, view_res=96, res=64, width=160)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    otree = oracle.tree_build(pts, res, dil)
    model = P.Model(tree, seed=1, ctx=ctx)
    om = oracle.init_model(otree, 1)
    st = P.RenderStats()
    rgb, a, d = P.render_frame(model, P.Camera.from_record(cam, W, H), stats=st)
    orgb, oa, od, ost = oracle.render_frame(otree, om, cam, W, H)
    assert ost[2] > 10 * W  # a non-trivial number of hits
    assert np.abs(rgb.reshape(-1) - orgb).max() <= 1e-5
    assert np.abs(d.reshape(-1) - od).max() <= 1e-5
    assert st.traversal_hits == ost[2] and st.rays_with_hits == ost[1]


def _psnr(a, b):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return 99.0 if mse == 0 else 10.0 * np.log10(1.0 / mse)


TOL_BF16_PSNR_DELTA = 0.05  # north_star: PSNR delta <= 0.05 dB with the bf16 MLP


@pytest.mark.parametrize("precision", ["bf16", "fp16"])
@pytest.mark.parametrize("objects", [4, 20])
def test_render_tensor_core(ctx, oracle, objects, precision):
    """tcgen05 16-bit decoder vs the fp32 oracle: PSNR(vs GT) delta <= 0.05 dB."""
    sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=objects, n_views=8, view_res=96, res=64, width=192)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    otree = oracle.tree_build(pts, res, dil)
    model = P.Model(tree, seed=1, ctx=ctx)
    om = oracle.init_model(otree, 1)
    st = P.RenderStats()
    rgb, a, d = P.render_frame(model, P.Camera.from_record(cam, W, H), stats=st, precision=precision)
    orgb, oa, od, ost = oracle.render_frame(otree, om, cam, W, H)
    gt, _, _ = S.render_gt(sc, cam, W, H)
    p16, p32, pv = _psnr(rgb.reshape(-1), gt), _psnr(orgb, gt), _psnr(rgb.reshape(-1), orgb)
    print(f"{precision} objects={objects} psnr_tc={p16:.4f} psnr_oracle={p32:.4f} psnr_bf16_vs_oracle={pv:.2f} "
          f"maxabs_rgb={np.abs(rgb.reshape(-1) - orgb).max():.3g} maxabs_depth={np.abs(d.reshape(-1) - od).max():.3g}")
    assert abs(p16 - p32) <= TOL_BF16_PSNR_DELTA
    assert pv > 40.0  # bf16 vs fp32 image agreement
    assert np.abs(a.reshape(-1) - oa).max() < 2e-2
    assert st.traversal_hits == ost[2]


@pytest.mark.parametrize("precision", ["bf16", "fp16"])
def test_render_tc_matches_fp32_path(c1, ctx, precision):
    tree, otree, cam, W, H = c1
    model = P.Model(tree, seed=1, ctx=ctx)
    camera = P.Camera.from_record(cam, W, H)
    r32, a32, d32 = P.render_frame(model, camera, precision="fp32")
    r16, a16, d16 = P.render_frame(model, camera, precision=precision)
    print(f"c1 {precision} vs fp32 psnr={_psnr(r16, r32):.2f} maxabs={np.abs(r16 - r32).max():.3g}")
    assert _psnr(r16, r32) > 40.0
    # depth = sum(w t_s) / alpha is ill-conditioned near the 1e-4 alpha cut; compare where alpha is material
    m = (a32 > 1e-2) & (a16 > 1e-2)
    assert m.sum() > 1000
    assert np.abs(d16 - d32)[m].max() < 5e-2


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_render_hit_buffer_overflow_retry(oracle, precision):
    """A fresh context sizes its hit buffers for ~4 hits/ray; a dense scene (~10 hits/ray,
    > 1M hits) overflows them on the first frame. The frame must be redone transparently
    (banded host path and device path), with no spurious geometry errors from the partial
    hit lists, and match the oracle."""
    pts = S.random_occupancy_points(32, 0.3, 5)
    W = 448
    cam = S.lookat_camera((0.5 + 1.8 * 0.6, 0.5 + 1.8 * 0.3, 0.5 + 1.8 * 0.7416), (0.5, 0.5, 0.5), W, W, 1.2 * W)
    otree = oracle.tree_build(pts, 32, 0)
    om = oracle.init_model(otree, 2)
    orgb, oa, od, ost = oracle.render_frame(otree, om, cam, W, W)
    assert ost[2] > (1 << 20) and ost[2] > 4 * W * W  # really overflows the initial capacity
    for fresh in range(2):  # first call overflows; second reuses the grown buffers
        c = P.Context(0)
        tree = P.SparseOctree.build(pts, P.GridConfig(32, dilation=0), c)
        model = P.Model(tree, seed=2, ctx=c)
        st = P.RenderStats()
        rgb, a, d = P.render_frame(model, P.Camera.from_record(cam, W, W), stats=st, precision=precision)
        assert st.traversal_hits == ost[2]
        tol = TOL_FP32 if precision == "fp32" else 2e-2
        assert np.abs(rgb.reshape(-1) - orgb).max() <= tol
        assert np.abs(a.reshape(-1) - oa).max() <= tol
        c.close()


@pytest.mark.parametrize("precision", ["fp16", "bf16", "fp32"])
def test_device_frame_submit_finish(precision):
    """svlf_render_frame_device_submit / _finish give the bits and RenderStats of
    svlf_render_frame_device, including a first frame that overflows a fresh context's hit
    buffers (the finish re-renders it); while a frame is pending the context refuses other
    work, and a finish without a submit is an error."""
    import torch

    pts = S.random_occupancy_points(32, 0.3, 5)
    W = 448
    cam = S.lookat_camera((0.5 + 1.8 * 0.6, 0.5 + 1.8 * 0.3, 0.5 + 1.8 * 0.7416), (0.5, 0.5, 0.5), W, W, 1.2 * W)
    camera = P.Camera.from_record(cam, W, W)
    bg = np.array([0.25, 0.5, 0.75], np.float32)
    n = W * W

    def bufs():
        return (torch.full((n * 3,), -1.0, device="cuda"), torch.full((n,), -1.0, device="cuda"),
                torch.full((n,), -1.0, device="cuda"))

    c = P.Context(0)
    tree = P.SparseOctree.build(pts, P.GridConfig(32, dilation=0), c)
    model = P.Model(tree, seed=2, ctx=c)
    got, gst = [], []
    for _ in range(2):  # the first submit overflows the initial hit capacity (> 1M hits)
        b, st = bufs(), P.RenderStats()
        P.render_frame_device_submit(model, camera, *(x.data_ptr() for x in b), background=bg,
                                     precision=precision)
        if not gst:
            with pytest.raises(Exception, match="pending"):
                P.render_frame_device(model, camera, *(x.data_ptr() for x in b), precision=precision)
        P.render_frame_device_finish(c, st)
        got.append(b)
        gst.append(st)
    with pytest.raises(Exception, match="no frame"):
        P.render_frame_device_finish(c)
    ref, rst = bufs(), P.RenderStats()
    P.render_frame_device(model, camera, *(x.data_ptr() for x in ref), stats=rst, background=bg,
                          precision=precision)
    torch.cuda.synchronize()
    assert rst.traversal_hits > (1 << 20)
    for b, st in zip(got, gst):
        for x, y in zip(b, ref):
            assert torch.equal(x, y)
        for f in ("rays", "rays_with_hits", "traversal_hits", "thickness_queries", "color_queries"):
            assert getattr(st, f) == getattr(rst, f)
    c.close()


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
@pytest.mark.parametrize("background", [None, (0.25, 0.5, 0.75)])
def test_host_frame_paths_agree(ctx, oracle, precision, background):
    """svlf_render_frame delivers the same bits through every host path: fresh pageable
    arrays, reused pageable buffers and page-locked buffers, synchronous (several bands)
    and submitted (one band) — and they are the bits of the device-buffer frame: the
    sparse transfer (foreground pixels + block table, background filled on the host)
    reproduces the composite's output exactly."""
    import torch

    sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=4, n_views=8, view_res=96, res=64, width=1280)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    model = P.Model(tree, seed=1, ctx=ctx)
    camera = P.Camera.from_record(cam, W, H)
    n = W * H
    dev = (torch.full((3 * n,), -1.0, device="cuda"), torch.full((n,), -1.0, device="cuda"),
           torch.full((n,), -1.0, device="cuda"))
    P.render_frame_device(model, camera, *(x.data_ptr() for x in dev), background=background, precision=precision)
    torch.cuda.synchronize()
    ref = [x.cpu().numpy() for x in dev]
    got = [x.reshape(-1).copy() for x in P.render_frame(model, camera, background=background, precision=precision)]
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)
    reuse = (np.full(3 * n, -1, np.float32), np.full(n, -1, np.float32), np.full(n, -1, np.float32))
    pinned = P.pinned_frame(W, H)
    for out in (reuse, pinned):
        for _ in range(2):
            P.render_frame(model, camera, background=background, precision=precision, out=out)
            for a, b in zip(out, ref):
                assert np.array_equal(a, b)
        P.render_frame_submit(model, camera, out, background=background, precision=precision).wait()
        for a, b in zip(out, ref):
            assert np.array_equal(a, b)
    assert ref[1].max() > 0.5  # the frame is not empty
    assert (ref[1] == 0).mean() > 0.3  # and has background


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_sparse_frame_estimate_exceeded(ctx, precision):
    """Sparse host frames copy as many foreground pixels as the previous frame of the band had
    (+1/8); a frame with far more foreground (the camera moved closer) takes the completion's
    extra copy. Every frame equals the device-buffer frame bit for bit, synchronous (several
    bands) and submitted (one band)."""
    import torch

    pts = S.random_occupancy_points(32, 0.3, 5)
    tree = P.SparseOctree.build(pts, P.GridConfig(32, dilation=0), ctx)
    model = P.Model(tree, seed=2, ctx=ctx)
    W = 1024  # several bands in the synchronous path
    n = W * W
    dev = (torch.empty(3 * n, device="cuda"), torch.empty(n, device="cuda"), torch.empty(n, device="cuda"))
    fgs = []
    for dist in (6.0, 1.8, 6.0, 1.5):  # far (little foreground), near (mostly foreground), ...
        cam = S.lookat_camera((0.5 + dist * 0.6, 0.5 + dist * 0.3, 0.5 + dist * 0.7416), (0.5, 0.5, 0.5), W, W,
                              1.2 * W)
        camera = P.Camera.from_record(cam, W, W)
        st = P.RenderStats()
        P.render_frame_device(model, camera, *(x.data_ptr() for x in dev), stats=st, background=(0.1, 0.2, 0.3),
                              precision=precision)
        torch.cuda.synchronize()
        ref = [x.cpu().numpy() for x in dev]
        fgs.append(st.rays_with_hits)
        got = P.render_frame(model, camera, background=(0.1, 0.2, 0.3), precision=precision)
        for a, b in zip(got, ref):
            assert np.array_equal(a.reshape(-1), b)
        out = P.pinned_frame(W, W)
        P.render_frame_submit(model, camera, out, background=(0.1, 0.2, 0.3), precision=precision).wait()
        for a, b in zip(out, ref):
            assert np.array_equal(a.reshape(-1), b)
    assert fgs[1] > 2 * fgs[0] and fgs[1] > n // 4  # the near frames exceed the far frames' estimate


def test_pipelined_frames(ctx, oracle):
    """render_frame_submit / wait: two frames in flight give the same bits and statistics as
    synchronous render_frame calls; a third submit is refused until a wait."""
    sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=4, n_views=8, view_res=96, res=64, width=640)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    model = P.Model(tree, seed=1, ctx=ctx)
    cams = S.hemisphere_cameras(2, 1.8, 11, W, H, 1.5 * W)
    cameras = [P.Camera.from_record(c, W, H) for c in cams]
    want, want_st = [], []
    for c in cameras:
        st = P.RenderStats()
        want.append([x.reshape(-1).copy() for x in P.render_frame(model, c, stats=st, precision="fp16")])
        want_st.append(st)
    frames = [P.pinned_frame(W, H), (np.empty(3 * W * H, np.float32), np.empty(W * H, np.float32),
                                     np.empty(W * H, np.float32))]  # page-locked and pageable
    for _ in range(2):
        t = [P.render_frame_submit(model, c, f, precision="fp16") for c, f in zip(cameras, frames)]
        with pytest.raises(ValueError):
            P.render_frame_submit(model, cameras[0], frames[0], precision="fp16")
        for k in range(2):
            st = P.RenderStats()
            got = t[k].wait(stats=st)
            for a, b in zip(got, want[k]):
                assert np.array_equal(a.reshape(-1), b)
            assert st.traversal_hits == want_st[k].traversal_hits and st.rays_with_hits == want_st[k].rays_with_hits


@pytest.mark.parametrize("res", [512, 1024])
def test_deep_octree_render_matches_oracle(ctx, oracle, res):
    """Octree depth 9-10 (C5-scale resolution): traversal hit lists bit-exact and the fp32
    render within 1e-3 of the oracle on a small frame of the RTMV-shaped scene."""
    sc = S.make_random_scene(7, 4)
    cams = S.hemisphere_cameras(12, 1.8, 7, 160, 160, 240.0)
    pts = S.occupancy_points(sc, cams, 160, 160)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=1), ctx)
    otree = oracle.tree_build(pts, res, 1)
    assert tree.leaf_level == otree.leaf_level and tree.vertex_count == otree.vertex_count
    W = 64
    cam = S.lookat_camera((0.5 + 1.8 * 0.6, 0.5 + 1.8 * 0.3, 0.5 + 1.8 * 0.7416), (0.5, 0.5, 0.5), W, W, 1.5 * W)
    rays = oracle.camera_rays(cam, W, W)
    _assert_hits_equal(tree.traverse(rays), oracle.traverse(otree, rays))
    model = P.Model(tree, seed=1, ctx=ctx)
    om = oracle.init_model(otree, 1)
    rgb, a, d = P.render_frame(model, P.Camera.from_record(cam, W, W), precision="fp32")
    orgb, oa, od, _ = oracle.render_frame(otree, om, cam, W, W)
    assert np.abs(rgb.reshape(-1) - orgb).max() <= TOL_FP32
    assert np.abs(d.reshape(-1) - od).max() <= TOL_FP32


@pytest.mark.parametrize("precision", ["fp16", "bf16", "fp32"])
def test_render_empty_and_tiny_frames(c1, oracle, ctx, precision):
    """Frames with no hit at all (camera facing away from the scene) and 1x1 / 3x2 frames through every
    decoder path: background and zero alpha/depth exactly like the reference."""
    tree, otree, cam, W, H = c1
    model = P.Model(tree, seed=2, ctx=ctx)
    om = oracle.init_model(otree, 2)
    away = S.lookat_camera((0.5, 0.5, 3.0), (0.5, 0.5, 6.0), 64, 48, 50.0)
    bg = np.array([0.25, 0.5, 0.75], np.float32)
    st = P.RenderStats()
    rgb, a, d = P.render_frame(model, P.Camera.from_record(away, 64, 48), background=bg, stats=st,
                               precision=precision)
    assert st.traversal_hits == 0 and st.rays_with_hits == 0
    assert np.array_equal(rgb.reshape(-1, 3), np.broadcast_to(bg, (64 * 48, 3)))
    assert not np.any(a) and not np.any(d)
    for w, h in ((1, 1), (3, 2)):
        c = S.lookat_camera(tuple(0.5 + 1.8 * x for x in S.C1_EYE_DIR), (0.5, 0.5, 0.5), w, h, 2.0)
        rgb, a, d = P.render_frame(model, P.Camera.from_record(c, w, h), precision=precision)
        orgb, oa, od, _ = oracle.render_frame(otree, om, c, w, h)
        tol = 1e-3 if precision == "fp32" else 3e-2
        assert np.abs(rgb.reshape(-1) - orgb).max() <= tol
        assert np.abs(a.reshape(-1) - oa).max() <= tol


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
@pytest.mark.parametrize("world", [2, 3])
def test_row_band_shards_stitch_to_the_full_frame(ctx, precision, world):
    """SURVEY.md §8(e) render sharding: each rank renders its row band (parallel.row_band) with
    svlf_render_rows_device; the stitched bands are bit-identical to the full frame (rays are
    independent, so band boundaries change nothing)."""
    import torch
    from paper_2205_07058_b200.parallel import row_band

    sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=4, n_views=8, view_res=96, res=64, width=160)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    model = P.Model(tree, seed=1, ctx=ctx)
    camera = P.Camera.from_record(cam, W, H)
    n = W * H

    def bufs():
        return (torch.zeros(n * 3, device="cuda"), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda"))

    full = bufs()
    P.render_frame_device(model, camera, *(b.data_ptr() for b in full), precision=precision)
    parts = bufs()
    for rank in range(world):
        r0, rows = row_band(H, rank, world)
        off = r0 * W
        P.render_frame_device(model, camera, parts[0][off * 3:].data_ptr(), parts[1][off:].data_ptr(),
                              parts[2][off:].data_ptr(), precision=precision, row0=r0, rows=rows)
    torch.cuda.synchronize()
    for a, b in zip(full, parts):
        assert torch.equal(a, b)
    assert float(full[1].sum()) > 0  # the frame has foreground


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
@pytest.mark.parametrize("world,tile", [(1, 32), (2, 16), (3, 32), (8, 8)])
def test_tile_interleaved_shards_stitch_to_the_full_frame(ctx, precision, world, tile):
    """one frame split across ranks as round-robin raster tiles
    (svlf_render_tiles_device); every rank's tiles, stitched, are bit-identical to the full frame,
    with RenderStats summing to the frame's. Round-robin tiles spread a clustered foreground over
    the ranks (the per-rank hit counts are reported)."""
    import torch
    from paper_2205_07058_b200.parallel import stitch_tiles

    sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=4, n_views=8, view_res=96, res=64, width=160)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    model = P.Model(tree, seed=1, ctx=ctx)
    camera = P.Camera.from_record(cam, W, H)
    n = W * H
    full = (torch.zeros(n * 3, device="cuda"), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda"))
    fst = P.RenderStats()
    P.render_frame_device(model, camera, *(b.data_ptr() for b in full), stats=fst, precision=precision)
    img = [np.zeros((H, W, 3), np.float32), np.zeros((H, W), np.float32), np.zeros((H, W), np.float32)]
    tot = P.RenderStats()
    hits = []
    for rank in range(world):
        k = P.tiles_owned(camera, tile, tile, rank, world)
        m = k * tile * tile
        b = (torch.zeros(max(m, 1) * 3, device="cuda"), torch.zeros(max(m, 1), device="cuda"),
             torch.zeros(max(m, 1), device="cuda"))
        st = P.RenderStats()
        P.render_tiles_device(model, camera, tile, tile, rank, world, *(x.data_ptr() for x in b), stats=st,
                              precision=precision)
        torch.cuda.synchronize()
        for dst, src in zip(img, b):
            stitch_tiles(dst, src[:m * (3 if dst.ndim == 3 else 1)].cpu().numpy(), W, H, tile, tile, rank, world)
        for f in ("rays", "rays_with_hits", "traversal_hits", "thickness_queries", "color_queries"):
            setattr(tot, f, getattr(tot, f) + getattr(st, f))
        hits.append(st.traversal_hits)
    print(f"world {world} tile {tile}: hits per rank {hits}")
    for a, b in zip(full, img):
        assert np.array_equal(a.cpu().numpy().reshape(b.shape), b)
    assert (tot.rays, tot.rays_with_hits, tot.traversal_hits) == (fst.rays, fst.rays_with_hits, fst.traversal_hits)
    with pytest.raises(ValueError):
        P.render_tiles_device(model, camera, 7, 7, 0, world, *(x.data_ptr() for x in full))
