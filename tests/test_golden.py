"""Pin the C restatement (oracle/svlf_oracle.c) to fixtures produced by the
unmodified reference (tests/golden/make_golden.py over oracle/_ref).

Bit-exact: octree codes/corner ids, traversal ids and t values, camera-frame
render (no-FMA reference build), Adam. Losses: identical to fp64 rounding
order; sampled gradients relative 1e-5 (the reference reduces weight
gradients with `omp simd` in an implementation-defined order)."""
import os

import numpy as np
import pytest

from oracle import Model

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(G, name))


def test_octree_c1(oracle):
    import paper_2205_07058_b200.synthetic as S

    g = _load("octree_c1.npz")
    pts, res, dil, *_ = S.c1_workload()
    t = oracle.tree_build(pts, res, dil)
    assert np.array_equal(t.leaf_codes, g["leaf_codes"])
    assert np.array_equal(t.corner_ids, g["corner_ids"])
    assert t.vertex_count == int(g["vertex_count"])
    assert [len(t.level_codes(l)) for l in range(t.leaf_level + 1)] == g["level_sizes"].tolist()


def test_traversal_reference_rays(oracle):
    import paper_2205_07058_b200.synthetic as S

    g = _load("traverse_rand16.npz")
    t = oracle.tree_build(S.random_occupancy_points(16, 0.1, 7), 16, 0)
    off, ids, tin, tout = oracle.traverse(t, g["rays"])
    assert np.array_equal(off, g["offsets"])
    assert np.array_equal(ids, g["ids"]) and np.array_equal(ids, g["ids_fma"])
    assert np.array_equal(tin, g["t_in"]) and np.array_equal(tout, g["t_out"])
    # the default (FMA-contracting) reference build agrees to ~1e-15
    assert np.abs(tin - g["t_in_fma"]).max() < 1e-12


def test_render_c1_64(oracle):
    import paper_2205_07058_b200.synthetic as S

    g = _load("render_c1_64.npz")
    pts, res, dil, *_ = S.c1_workload()
    t = oracle.tree_build(pts, res, dil)
    m = oracle.init_model(t, 1)
    assert np.array_equal(m.ft[:256], g["init_ft_head"]) and np.array_equal(m.mt[:256], g["init_mt_head"])
    assert np.array_equal(m.mc[-256:], g["init_mc_tail"])
    rgb, a, d, st = oracle.render_frame(t, m, g["camera"], 64, 64)
    assert np.array_equal(rgb, g["rgb"]) and np.array_equal(a, g["alpha"]) and np.array_equal(d, g["depth"])
    assert st.tolist() == g["stats"].tolist()
    assert np.abs(rgb - g["rgb_fma"]).max() < 1e-6


@pytest.mark.parametrize("tag,mode,frozen,lw", [("surf", 0, False, (1.0, 0.01, 0.01, 0.1)),
                                                ("surf0", 0, False, (1.0, 0.01, 0.0, 0.1)),
                                                ("vol", 1, False, (1.0, 0.01, 0.01, 0.1)),
                                                ("volfz", 1, True, (1.0, 0.01, 0.01, 0.1))])
def test_losses_and_gradients(oracle, tag, mode, frozen, lw):
    g = _load("loss_small.npz")
    t = oracle.tree_build(g["occ_points"], 16, 1)
    m = oracle.init_model(t, 0)
    loss, gr, st = oracle.loss(t, m, g["rays"], g["c_gt"], g["depth"], g["alpha"], mode, lw=lw, frozen=frozen)
    assert loss == pytest.approx(float(g[f"{tag}_loss"]), rel=1e-12)
    assert st.tolist() == g[f"{tag}_stats"].tolist()
    for k in ("ft", "fc", "mt", "mc"):
        arr = getattr(gr, k)
        assert np.linalg.norm(arr.astype(np.float64)) == pytest.approx(float(g[f"{tag}_{k}_norm"]), rel=1e-5, abs=1e-30)
        np.testing.assert_allclose(arr[g[f"{tag}_{k}_idx"]], g[f"{tag}_{k}_val"], rtol=1e-4, atol=1e-9)


def test_adam(oracle):
    g = _load("adam.npz")
    p, m, v = g["p0"].copy(), np.zeros(1000, np.float32), np.zeros(1000, np.float32)
    oracle.adam_step(p, g["g1"], m, v, 0, np.float32(1e-3))
    oracle.adam_step(p, g["g2"], m, v, 1, np.float32(1e-3))
    assert np.array_equal(p, g["p"]) and np.array_equal(m, g["m"]) and np.array_equal(v, g["v"])
