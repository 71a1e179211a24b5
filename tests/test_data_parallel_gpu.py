"""Data-parallel train step of the library with world = 2.

Two processes (tests/dp_worker.py) each step their own half of the image
(contiguous row bands: their touched feature rows differ) through
svlf_train_step with the exchange attached (host-staged all-reduce over
torch.distributed gloo). This runs the library's whole exchange -- the loss /
statistics reduction, the dense decoder all-reduce and the sparse feature
path (touched-row flags, max all-reduce, compaction, pack, sum, scatter) --
with ranks whose touched sets differ. Gates: the exchanged gradients equal
the full batch's gradients (reference semantics: gradients are sums over
rays, src/train.cpp:473-478); both ranks hold bit-identical parameters after
two steps; those equal a single-rank full-batch run up to rounding.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2205_07058_b200 as P

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import dp_worker  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_two_rank_exchange_matches_full_batch(tmp_path, precision):
    port = str(_free_port())
    outs = [str(tmp_path / f"r{r}.npz") for r in range(2)]
    env = dict(os.environ, PYTHONPATH=os.path.dirname(HERE))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dp_worker.py"), str(r), "2", port, outs[r],
                               precision], env=env) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    r0, r1 = (dict(np.load(o)) for o in outs)

    # full batch on one context, no collective
    pts, res, W, rays, cgt, depth, alpha = dp_worker.scene()
    ctx = P.Context(0)
    ctx.set_train_precision(precision)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=1), ctx)
    model = P.Model(tree, seed=0, ctx=ctx)
    st = P.LossStats()
    loss = P.loss_grads(model, rays, cgt, depth, alpha, mode="volumetric", stats=st)
    full_g = model.get_grads()
    model = P.Model(tree, seed=0, ctx=ctx)
    losses = [P.train_step(model, rays, cgt, depth, alpha, mode="surface", lr=1e-3),
              P.train_step(model, rays, cgt, depth, alpha, mode="volumetric", lr=1e-3)]
    full_p = model.get_params()

    # the two shards touch different feature rows, so the sparse path really merges two sets
    corners = tree.corner_ids().reshape(-1, 8)
    leaf_index = {int(c): i for i, c in enumerate(tree.leaf_codes)}
    touched = []
    for r in range(2):
        ids = tree.traverse(rays[dp_worker.shard_of(W, W, r, 2)])[1]
        touched.append({int(v) for c in set(ids.tolist()) for v in corners[leaf_index[c]]})
    assert touched[0] - touched[1] and touched[1] - touched[0]

    for r in (r0, r1):
        assert abs(r["grad_loss"] - loss) <= 1e-9 * abs(loss)  # the all-reduced loss is the full sum
        assert r["grad_stats"].tolist() == [st.rays, st.skipped_rays, st.eta_skipped]
        tol = 1e-5 if precision == "fp32" else 2e-2
        for k, g in zip(("g_ft", "g_fc", "g_mt", "g_mc"), full_g):
            assert _rel_l2(r[k], g) <= tol, (k, _rel_l2(r[k], g))
    # replicated parameters stay bit-identical across ranks
    for k in ("p_ft", "p_fc", "p_mt", "p_mc"):
        assert np.array_equal(r0[k], r1[k]), k
    assert r0["steps"].tolist() == [2] * 14
    np.testing.assert_allclose(r0["losses"], losses, rtol=1e-6)
    for k, p in zip(("p_ft", "p_fc", "p_mt", "p_mc"), full_p):
        d = np.abs(r0[k] - p)
        assert np.mean(d > 1e-6) < 5e-3, k  # Adam's first steps amplify rounding-level gradient differences
        assert d.max() <= 2.5e-3, k
    del model, tree
    ctx.close()
