"""Parity on the configurations the bench times (BASELINE.json configs 2 and 3).

* C2: the full 1600x1600 frame of the RTMV-shaped 4-object scene (octree depth
  8 from 100 hemisphere depth maps, init_model seed 1) rendered by the
  reference itself (oracle/_ref, its own build flags, all host threads) and by
  the GPU: fp32 max-abs <= 1e-3 (north_star) with identical RenderStats; the
  fp16 / bf16 tensor-core frames against the same reference frame.
* Trained model: svlf::train (the C++ stage driver over the GPU train step)
  trains a model; the validation view rendered by the GPU in fp32 / fp16 /
  bf16 and by the reference (same parameters) is scored against the analytic
  ground truth: PSNR delta <= 0.05 dB (north_star's bf16 gate), with weights
  that have moved away from their initialisation.
* C3: the 2^18-ray train step (depth 8): loss and gradients against the
  reference's own loss + backward (ref_loss = the public surface_loss /
  volumetric_loss summed over the batch) in both stage modes.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _psnr(a, b):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10 * np.log10(1.0 / mse)


def _rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


@pytest.fixture(scope="module")
def ctx():
    c = P.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def c2(ctx, reference):
    sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=4, ctx=ctx)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    model = P.Model(tree, seed=1, ctx=ctx)
    rt = reference.tree_build(pts, res, dil)
    rm = reference.init_model(rt, 1)
    rgb, alpha, depth, st = reference.render_frame(rt, rm, cam, W, H)
    return tree, model, P.Camera.from_record(cam, W, H), (rgb, alpha, depth), st


def test_c2_fp32_frame_matches_reference(c2):
    tree, model, cam, (rgb, alpha, depth), rst = c2
    st = P.RenderStats()
    g = P.render_frame(model, cam, stats=st, precision="fp32")
    errs = [float(np.abs(a.reshape(-1) - b).max()) for a, b in zip(g, (rgb, alpha, depth))]
    print("C2 fp32 max-abs rgb/alpha/depth", errs, "hits", st.traversal_hits)
    assert [st.rays, st.rays_with_hits, st.traversal_hits, st.thickness_queries, st.color_queries] == rst.tolist()
    assert max(errs) <= 1e-3


@pytest.mark.parametrize("precision", ["fp16", "bf16"])
def test_c2_tensor_core_frame_against_reference(c2, precision):
    """The timed configuration itself. Gates at the observed level: image PSNR against the
    reference frame (fp16: 10-bit mantissa operands, bf16: 7-bit), alpha and depth max-abs."""
    tree, model, cam, (rgb, alpha, depth), rst = c2
    st = P.RenderStats()
    g = P.render_frame(model, cam, stats=st, precision=precision)
    p = _psnr(g[0].reshape(-1), rgb)
    ea, ed = float(np.abs(g[1].reshape(-1) - alpha).max()), float(np.abs(g[2].reshape(-1) - depth).max())
    print(f"C2 {precision}: PSNR vs reference {p:.2f} dB, alpha max-abs {ea:.3g}, depth max-abs {ed:.3g}")
    assert [st.rays, st.rays_with_hits, st.traversal_hits, st.thickness_queries, st.color_queries] == rst.tolist()
    assert p >= (75.0 if precision == "fp16" else 60.0)
    assert ea <= (2e-3 if precision == "fp16" else 1e-2)


@pytest.fixture(scope="module")
def trained(tmp_path_factory, reference):
    """A model trained by svlf::train (tests/cpp/cpp_api_probe trainloop: the C++ stage driver over
    the GPU train step) on 24 views of make_random_scene(7, 4) at 96^2, 4 of them validation."""
    d = tmp_path_factory.mktemp("trained")
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    W, n = 96, 24
    scene = reference.scene_make(7, 4)
    cams = reference.hemisphere_cameras(n, 1.8, 7, W, W, 1.5 * W)
    splits = np.array([1 if k % 6 == 5 else 0 for k in range(n)], np.int32)
    with open(d / "ds.bin", "wb") as f:
        f.write(np.array([n, W, W], np.uint32).tobytes())
        for k in range(n):
            rgb, depth, mask = reference.scene_render_gt(scene, cams[k], W, W)
            f.write(cams[k].astype(np.float64).tobytes())
            f.write(np.array([splits[k]], np.int32).tobytes())
            for a in (rgb, depth, mask):
                f.write(np.ascontiguousarray(a, np.float32).tobytes())
    r = subprocess.run([os.path.join(ROOT, "build", "cpp_tests", "cpp_api_probe"), "trainloop", str(d), "8", "8",
                        "8", "64"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    log = np.fromfile(d / "train_log.f64", np.float64).reshape(-1, 5)
    meta = np.fromfile(d / "tree_meta.u32", np.uint32)
    codes = np.fromfile(d / "leaf_codes.u64", np.uint64)
    flat = np.fromfile(d / "trained.f32", np.float32)
    return scene, cams, splits, W, log, meta, codes, flat


def test_trained_model_psnr_delta(ctx, trained, reference):
    scene, cams, splits, W, log, meta, codes, flat = trained
    res, dil, V = int(meta[0]), int(meta[1]), int(meta[2])
    a, b = V * 64, V * 96
    parts = (flat[:a], flat[a:b], flat[b:b + P.DEC_T_SIZE], flat[b + P.DEC_T_SIZE:])
    tree = P.SparseOctree.from_leaves(codes, P.GridConfig(res, dilation=dil), ctx)
    model = P.Model(tree, ctx=ctx)
    model.set_params(*parts)
    init = P.Model(tree, seed=0, ctx=ctx).get_params()
    moved = _rel_l2(parts[3], init[3])
    assert moved > 0.05  # the decoders really trained (not the initialisation)
    rt = reference.tree_from_leaves(codes, res, dil)
    import oracle as O

    rm = O.Model(*[np.ascontiguousarray(x) for x in parts])
    R = 256  # validation views rendered at a higher resolution than trained
    for k in np.flatnonzero(splits == 1)[:2]:
        cam = np.array(cams[k], np.float64).copy()
        cam[:4] *= R / W  # fx fy cx cy scale with the resolution
        gt = reference.scene_render_gt(scene, cam, R, R)[0].reshape(-1)
        ref = reference.render_frame(rt, rm, cam, R, R)[0]
        camera = P.Camera.from_record(cam, R, R)
        p_ref = _psnr(ref, gt)
        out = {}
        for prec in ("fp32", "fp16", "bf16"):
            img = P.render_frame(model, camera, precision=prec)[0].reshape(-1)
            out[prec] = (_psnr(img, gt), _psnr(img, ref), float(np.abs(img - ref).max()))
        print(f"view {k}: PSNR(ref, gt) {p_ref:.3f} dB;",
              {p: tuple(round(x, 4) for x in v) for p, v in out.items()}, "final train loss", log[-1, 2])
        assert p_ref > 12.0  # a trained model, not noise
        assert out["fp32"][2] <= 1e-3
        for prec in ("fp16", "bf16"):
            assert abs(out[prec][0] - p_ref) <= 0.05, prec
        assert out["fp16"][1] >= 60.0 and out["bf16"][1] >= 45.0


@pytest.fixture(scope="module")
def c3(ctx, reference_nofma, reference):
    sc, cam, pts, res, dil, rays, cgt, depth, alpha = S.c3_workload()
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
    alpha = alpha.astype(np.uint8)
    refs = {}
    for mode in ("volumetric", "surface"):
        m = 0 if mode == "surface" else 1
        out = []
        for R in (reference_nofma, reference):  # the reference without and with its default FMA contraction
            rt = R.tree_build(pts, res, dil)
            out.append(R.loss(rt, R.init_model(rt, 0), rays, cgt, depth, alpha, m))
        refs[mode] = out
    return tree, rays, cgt, depth, alpha, refs


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("mode", ["volumetric", "surface"])
def test_c3_train_step_matches_reference(ctx, c3, mode, precision):
    """The bench's C3 train step (2^18 rays, depth 8): loss and gradients against the reference
    (no-FMA build) at the fp32 gates (loss 1e-6 rel, gradients 1e-4 rel-L2) or the 16-bit gates
    (tf32: 1e-3, 2e-2). At this size a rounding-level change of the forward pass moves a few
    hits across a relu / tau > 0 boundary: the reference's own two builds (with and without
    FMA contraction) differ by `floor` per tensor (1.4e-4 on feat_t, all of it in one row
    group), and the fp32 gate is max(1e-4, 2 x floor); a feature tensor may instead show such a
    concentrated flip of its own (<= 5e-3) when the rest of it (all but the worst 0.1 % of
    rows) meets 1e-4."""
    tree, rays, cgt, depth, alpha, refs = c3
    ctx.set_train_precision(precision)
    try:
        model = P.Model(tree, seed=0, ctx=ctx)
        st = P.LossStats()
        loss = P.loss_grads(model, rays, cgt, depth, alpha, mode=mode, stats=st)
        g = model.get_grads()
    finally:
        ctx.set_train_precision("fp32")
    (rloss, rg, rst), (floss, fg, _) = refs[mode]
    names = ("ft", "fc", "mt", "mc")
    errs = [_rel_l2(a, getattr(rg, k)) for a, k in zip(g, names)]
    floor = [_rel_l2(getattr(fg, k), getattr(rg, k)) for k in names]
    # A discrete event (a hit whose relu / tau > 0 / eta decision flips at rounding level) shows up
    # as an error concentrated in a handful of feature rows; bulk_err excludes the worst 0.1 % of rows.
    def bulk(a, b, w):
        d = np.linalg.norm((a - b).reshape(-1, w), axis=1)
        keep = np.argsort(d)[: d.size - max(1, d.size // 1000)]
        ref = b.reshape(-1, w)[keep]
        return float(np.linalg.norm(d[keep]) / max(np.linalg.norm(ref), 1e-30))

    bulk_errs = (bulk(g[0], rg.ft, 64), bulk(g[1], rg.fc, 32))
    fma_errs = [_rel_l2(a, getattr(fg, k)) for a, k in zip(g, names)]
    print(f"C3 {mode} {precision}: loss rel {abs(loss - rloss) / abs(rloss):.3g}, grad rel-L2 {errs} "
          f"(vs the FMA build {fma_errs}), reference FMA-vs-noFMA {floor}, "
          f"feature-gradient rel-L2 outside the worst 0.1% rows (t, c) {bulk_errs}")
    assert [st.rays, st.skipped_rays, st.eta_skipped] == list(rst)
    if precision == "fp32":
        assert abs(loss - rloss) <= 1e-6 * abs(rloss)
        for k, (e, f) in enumerate(zip(errs, floor)):
            if e <= max(1e-4, 2 * f):
                continue
            # only a concentrated (flip-type) difference in a feature tensor is tolerated, and the
            # rest of that tensor must meet the fp32 gate
            assert k < 2 and e <= 5e-3 and bulk_errs[k] <= 1e-4, (names[k], e, bulk_errs[k])
    else:
        assert abs(loss - rloss) <= 1e-3 * abs(rloss)
        assert max(errs) <= 2e-2


def test_step_buffers_grow_and_rerun(c3):
    """A context whose per-hit matrices were sized by a small batch (65,536 active hits) gets the
    2^18-ray C3 batch (~154 K active hits): the step detects the overflow on the device, skips its
    update, grows the buffers and re-runs (new graph capture); the result equals a fresh context's."""
    tree, rays, cgt, depth, alpha, refs = c3
    fresh, small = P.Context(0), P.Context(0)
    t_f = P.SparseOctree.from_leaves(tree.leaf_codes, tree.config, fresh)
    t_s = P.SparseOctree.from_leaves(tree.leaf_codes, tree.config, small)
    m_f, m_s = P.Model(t_f, seed=0, ctx=fresh), P.Model(t_s, seed=0, ctx=small)
    P.loss_grads(m_s, rays[:4096], cgt[:4096], depth[:4096], alpha[:4096], mode="volumetric")
    l_s = P.train_step(m_s, rays, cgt, depth, alpha, mode="volumetric", lr=1e-3)
    l_f = P.train_step(m_f, rays, cgt, depth, alpha, mode="volumetric", lr=1e-3)
    assert l_s == l_f
    assert m_s.get_adam()[2].tolist() == [1] * 14  # exactly one update despite the re-run
    for a, b in zip(m_s.get_params(), m_f.get_params()):
        d = np.abs(a - b)
        assert np.mean(d > 1e-6) < 1e-3 and d.max() <= 2.5e-3
    del m_s, m_f, t_s, t_f
    fresh.close()
    small.close()
