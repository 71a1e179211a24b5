"""GPU parity of the train step (loss, gradients, Adam) vs the CPU oracle.

Gradient oracle: the reference's public per-ray
surface_loss / volumetric_loss summed over the batch, restated in
oracle/svlf_oracle.c (pinned against the reference by test_oracle_vs_ref.py).
Tolerances: loss sum relative 1e-6 (fp32 forward whose dense layers run as
GEMMs, so the k summation order differs from the reference's; loss math is
fp64); gradients relative L2 <= 1e-4 per tensor (fp32; GEMM order and atomics
reorder the sums); Adam: parameters within one step size after two steps.
"""
import numpy as np
import pytest

import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S

pytestmark = pytest.mark.gpu

GRAD_REL_L2 = 1e-4
LOSS_REL = 1e-6  # fp32 forward (dense layers as GEMMs: k summation order differs from the reference)


@pytest.fixture(scope="module")
def ctx():
    c = P.Context(0)
    yield c
    c.close()


def _scene(W=48, res=32, frames=3, prims=4, seed=7):
    sc = S.make_random_scene(seed, prims)
    cams = S.hemisphere_cameras(frames, 1.8, seed, W, W, 1.5 * W)
    pts = S.occupancy_points(sc, cams, W, W)
    rgb, depth, mask = S.render_gt(sc, cams[0], W, W)
    rays = S.camera_rays(cams[0], W, W)
    return pts, res, rays, rgb.reshape(-1, 3), depth.astype(np.float64), (mask > 0.5).astype(np.uint8)


@pytest.fixture(scope="module")
def batch(ctx, oracle):
    pts, res, rays, cgt, depth, alpha = _scene()
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=1), ctx)
    otree = oracle.tree_build(pts, res, 1)
    return tree, otree, rays, cgt, depth, alpha


def _rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


MODES = [("surface", False, (1.0, 0.01, 0.01, 0.1)),
         ("surface", False, (1.0, 0.01, 0.0, 0.1)),   # lambda_empty = 0: surface voxel only
         ("volumetric", False, (1.0, 0.01, 0.01, 0.1)),
         ("volumetric", True, (1.0, 0.01, 0.01, 0.1))]


@pytest.fixture(scope="module")
def ctx_x3():
    c = P.Context(0)
    c.set_train_precision("tf32x3")
    yield c
    c.close()


@pytest.mark.parametrize("precision", ["fp32", "tf32x3"])
@pytest.mark.parametrize("mode,frozen,lw", MODES)
def test_loss_and_gradients_match_oracle(batch, ctx, ctx_x3, oracle, mode, frozen, lw, precision):
    """fp32 gates (loss 1e-6 relative, gradients 1e-4 rel-L2 per tensor) for the 3xTF32 split-operand
    tensor-core GEMMs ('fp32' and 'tf32x3' are the same arithmetic; both names are accepted)."""
    tree, otree, rays, cgt, depth, alpha = batch
    if precision == "tf32x3":
        ctx = ctx_x3
        tree = P.SparseOctree.from_leaves(tree.leaf_codes, tree.config, ctx)
    model = P.Model(tree, seed=0, ctx=ctx)
    om = oracle.init_model(otree, 0)
    st = P.LossStats()
    loss = P.loss_grads(model, rays, cgt, depth, alpha, mode=mode, color_frozen=frozen,
                        weights=P.LossWeights(*lw), stats=st)
    oloss, og, ost = oracle.loss(otree, om, rays, cgt, depth, alpha, 0 if mode == "surface" else 1, lw=lw,
                                 frozen=frozen)
    g = model.get_grads()
    print(precision, mode, frozen, "loss rel", abs(loss - oloss) / abs(oloss),
          [_rel_l2(a, b) for a, b in zip(g, (og.ft, og.fc, og.mt, og.mc))])
    assert abs(loss - oloss) <= LOSS_REL * abs(oloss)
    assert [st.rays, st.skipped_rays, st.eta_skipped] == list(ost)
    for name, a, b in zip(("feat_t", "feat_c", "dec_t", "dec_c"), g, (og.ft, og.fc, og.mt, og.mc)):
        if frozen and name in ("feat_c", "dec_c"):
            assert not np.any(a), name  # colour frozen: exactly zero
            continue
        assert _rel_l2(a, b) <= GRAD_REL_L2, (name, _rel_l2(a, b))


def test_adam_step_matches_oracle(batch, ctx, oracle):
    tree, otree, rays, cgt, depth, alpha = batch
    model = P.Model(tree, seed=0, ctx=ctx)
    om = oracle.init_model(otree, 0)
    lr = np.float32(1e-3)
    for step in range(2):
        P.train_step(model, rays, cgt, depth, alpha, mode="volumetric", lr=float(lr))
        _, og, _ = oracle.loss(otree, om, rays, cgt, depth, alpha, 1)
        if step == 0:
            ms = {k: np.zeros_like(getattr(om, k)) for k in ("ft", "fc", "mt", "mc")}
            vs = {k: np.zeros_like(getattr(om, k)) for k in ("ft", "fc", "mt", "mc")}
        for k in ("ft", "fc", "mt", "mc"):
            # per-tensor Adam over the flat layout (every tensor is at the same step here)
            oracle.adam_step(getattr(om, k), getattr(og, k), ms[k], vs[k], step, lr)
    got = model.get_params()
    for name, a, b in zip(("feat_t", "feat_c", "dec_t", "dec_c"), got, (om.ft, om.fc, om.mt, om.mc)):
        # Adam's first steps move every element by ~lr * sign(g); a gradient that is zero to
        # rounding can flip sign, so compare with a bound of one step size on those elements
        diff = np.abs(a - b)
        assert np.mean(diff > 1e-6) < 1e-3, name
        assert diff.max() <= 2.5 * lr, name
    m, v, steps = model.get_adam()
    assert steps.tolist() == [2] * 14


def test_adam_bit_exact_on_the_step_gradients(batch, ctx, oracle):
    """k_adam against the oracle's adam_step (src/mlp.cpp:277-296, pinned bit-exact to the no-FMA
    reference) on the gradients the step itself computed: parameters, m and v bit-identical after each
    of three steps (fresh and non-zero moments)."""
    tree, otree, rays, cgt, depth, alpha = batch
    model = P.Model(tree, seed=0, ctx=ctx)
    lr = np.float32(1e-3)
    p = [x.copy() for x in model.get_params()]
    m = [np.zeros_like(x) for x in p]
    v = [np.zeros_like(x) for x in p]
    for step in range(3):
        P.train_step(model, rays, cgt, depth, alpha, mode="volumetric", lr=float(lr))
        for i, g in enumerate(model.get_grads()):
            oracle.adam_step(p[i], g, m[i], v[i], step, lr)
        got = model.get_params()
        gm, gv, steps = model.get_adam()
        off = 0
        for i in range(4):
            assert np.array_equal(got[i], p[i]), (step, i)
            assert np.array_equal(gm[off:off + p[i].size], m[i]) and np.array_equal(gv[off:off + p[i].size], v[i])
            off += p[i].size
        assert steps.tolist() == [step + 1] * 14


def test_adam_hyperparameters_are_per_tensor(batch, ctx, oracle):
    """AdamState beta1/beta2/eps are honoured per tensor (mlp.hpp:117-128), not hard-coded."""
    tree, otree, rays, cgt, depth, alpha = batch
    model = P.Model(tree, seed=0, ctx=ctx)
    b1, b2, eps = model.get_adam_hyper()
    assert np.allclose(b1, 0.9) and np.allclose(b2, 0.999) and np.allclose(eps, 1e-8)
    nb1, neps = np.full(14, 0.8, np.float32), np.full(14, 1e-3, np.float32)
    model.set_adam_hyper(nb1, b2, neps)
    p0 = [x.copy() for x in model.get_params()]
    P.train_step(model, rays, cgt, depth, alpha, mode="volumetric", lr=1e-3)
    g = model.get_grads()
    got = model.get_params()
    # first step: mh = g, vh = g^2 (bias-corrected), so p -= lr g / (|g| + eps); eps = 1e-3 makes it
    # differ from the default eps = 1e-8 wherever |g| is not >> 1e-3
    gd = g[0].astype(np.float64)
    ft = p0[0].astype(np.float64) - np.float64(np.float32(1e-3)) * gd / (np.abs(gd) + np.float64(neps[0]))
    assert np.max(np.abs(got[0] - ft.astype(np.float32))) <= 2e-8
    default = p0[0].astype(np.float64) - np.float64(np.float32(1e-3)) * gd / (np.abs(gd) + np.float64(np.float32(1e-8)))
    assert np.max(np.abs(got[0] - default.astype(np.float32))) > 1e-5
    assert model.get_adam_hyper()[0][0] == np.float32(0.8)


def test_decoder_gradients_reproducible(batch, ctx):
    """Weight gradients are reduced in a fixed CTA order (no atomics): two identical calls give
    bit-identical decoder gradients."""
    tree, otree, rays, cgt, depth, alpha = batch
    model = P.Model(tree, seed=0, ctx=ctx)
    P.loss_grads(model, rays, cgt, depth, alpha, mode="volumetric")
    a = model.get_grads()
    P.loss_grads(model, rays, cgt, depth, alpha, mode="volumetric")
    b = model.get_grads()
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])


def test_train_step_reduces_loss(batch, ctx):
    tree, otree, rays, cgt, depth, alpha = batch
    model = P.Model(tree, seed=0, ctx=ctx)
    losses = [P.train_step(model, rays, cgt, depth, alpha, mode="surface", lr=1e-2) for _ in range(30)]
    assert losses[-1] < 0.8 * losses[0]


def test_frozen_stage_keeps_color_parameters(batch, ctx):
    tree, otree, rays, cgt, depth, alpha = batch
    model = P.Model(tree, seed=0, ctx=ctx)
    before = model.get_params()
    P.train_step(model, rays, cgt, depth, alpha, mode="volumetric", color_frozen=True, lr=1e-3)
    after = model.get_params()
    assert np.array_equal(before[1], after[1]) and np.array_equal(before[3], after[3])
    assert not np.array_equal(before[0], after[0]) and not np.array_equal(before[2], after[2])
    steps = model.get_adam()[2]
    assert steps[0] == 1 and steps[1] == 0 and list(steps[2:6]) == [1] * 4 and list(steps[6:]) == [0] * 8


@pytest.mark.parametrize("precision", ["fp32", "tf32x3"])
def test_nccl_attached_single_rank_matches_local(batch, oracle, precision):
    """Data-parallel path with a 1-rank NCCL communicator: the all-reduced step must equal the
    local step (loss identical, parameters identical up to atomic-order rounding)."""
    tree, otree, rays, cgt, depth, alpha = batch
    a, b = P.Context(0), P.Context(0)
    a.set_train_precision(precision)
    b.set_train_precision(precision)
    b.attach_nccl(P.nccl_unique_id(), 0, 1)
    codes = tree.leaf_codes
    ta = P.SparseOctree.from_leaves(codes, tree.config, a)
    tb = P.SparseOctree.from_leaves(codes, tree.config, b)
    ma, mb = P.Model(ta, seed=0, ctx=a), P.Model(tb, seed=0, ctx=b)
    for _ in range(2):
        la = P.train_step(ma, rays, cgt, depth, alpha, mode="volumetric", lr=1e-3)
        lb = P.train_step(mb, rays, cgt, depth, alpha, mode="volumetric", lr=1e-3)
        assert abs(la - lb) <= LOSS_REL * abs(la)
    share = 1e-3  # feature-gradient scatters use fp32 atomics: rounding-level differences
    for x, y in zip(ma.get_params(), mb.get_params()):
        assert np.mean(np.abs(x - y) > 1e-6) < share
        assert np.abs(x - y).max() <= 2.5e-3
    assert mb.get_adam()[2].tolist() == [2] * 14
    b.detach_nccl()


@pytest.mark.parametrize("mode,frozen,lw", MODES)
def test_tf32_train_mode_within_16bit_tolerance(batch, oracle, mode, frozen, lw):
    """TF32 mode (weight-gradient GEMMs on tensor cores): loss within 1e-3 relative and gradients within
    rel-L2 2e-2 per tensor of the oracle (SURVEY.md §8(c) 16-bit-mode gates)."""
    tree, otree, rays, cgt, depth, alpha = batch
    c = P.Context(0)
    c.set_train_precision("tf32")
    t = P.SparseOctree.from_leaves(tree.leaf_codes, tree.config, c)
    model = P.Model(t, seed=0, ctx=c)
    om = oracle.init_model(otree, 0)
    st = P.LossStats()
    loss = P.loss_grads(model, rays, cgt, depth, alpha, mode=mode, color_frozen=frozen,
                        weights=P.LossWeights(*lw), stats=st)
    oloss, og, ost = oracle.loss(otree, om, rays, cgt, depth, alpha, 0 if mode == "surface" else 1, lw=lw,
                                 frozen=frozen)
    assert abs(loss - oloss) <= 1e-3 * abs(oloss)
    assert [st.rays, st.skipped_rays, st.eta_skipped] == list(ost)
    for name, a, b in zip(("feat_t", "feat_c", "dec_t", "dec_c"), model.get_grads(), (og.ft, og.fc, og.mt, og.mc)):
        if frozen and name in ("feat_c", "dec_c"):
            assert not np.any(a), name
            continue
        assert _rel_l2(a, b) <= 2e-2, (name, _rel_l2(a, b))
    with pytest.raises(ValueError):
        c.set_train_precision("fp16")
    del model, t
    c.close()


def _pin(a):
    p = P.pinned_empty(a.size, a.dtype)
    p[:] = a.reshape(-1)
    return p.reshape(a.shape)


@pytest.mark.parametrize("pinned", [False, True])
def test_pipelined_steps_match_sequential_steps(batch, ctx, pinned):
    """TrainPipeline (svlf_train_batch_stage / svlf_train_step_staged: batch k + 1 uploaded while
    step k runs) gives the same losses and parameters as train_step batch by batch, from pageable
    (background staging thread) and page-locked (direct DMA) arrays."""
    tree, otree, rays, cgt, depth, alpha = batch
    n = rays.shape[0]
    rng = np.random.default_rng(1)
    batches = []
    for k in range(4):  # different sizes and orders, so a stale slot would show
        idx = np.tile(rng.permutation(n)[: n - 97 * k], 30)  # ~65K rays: chunked, pool-parallel staging
        b = [np.ascontiguousarray(x[idx]) for x in (rays, cgt.astype(np.float32), depth, alpha)]
        batches.append([_pin(x) for x in b] if pinned else b)
    m1 = P.Model(tree, seed=0, ctx=ctx)
    seq = [P.train_step(m1, *b, mode="volumetric", lr=1e-3) for b in batches]
    m2 = P.Model(tree, seed=0, ctx=ctx)
    pipe = P.TrainPipeline(m2)
    pipe.stage(*batches[0])
    got = []
    for k in range(len(batches)):
        if k + 1 < len(batches):
            pipe.stage(*batches[k + 1])
        got.append(pipe.step(mode="volumetric", lr=1e-3))
    assert got[0] == seq[0]  # same model, same batch: the forward and loss are deterministic
    np.testing.assert_allclose(got, seq, rtol=1e-6)  # later steps: feature-gradient atomics reorder sums
    for a, b in zip(m1.get_params(), m2.get_params()):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-6)
    # two slots: a third staged batch is refused until one is stepped or discarded
    pipe.stage(*batches[0])
    pipe.stage(*batches[1])
    with pytest.raises(ValueError, match="staging slots"):
        pipe.stage(*batches[2])
    pipe.drain()
    assert len(pipe) == 0
    with pytest.raises(ValueError, match="no batch staged"):
        pipe.step()
    pipe.stage(*batches[2])
    assert np.isfinite(pipe.step(mode="volumetric", lr=1e-3))
