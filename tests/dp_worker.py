"""One rank of the data-parallel train-step test (tests/test_data_parallel_gpu.py).

Runs the library's data-parallel step (svlf_train_step with a collective
attached: loss/statistics and decoder gradients all-reduced densely, feature
gradients through the touched-row union / pack / all-reduce / scatter of
train.cu) on this rank's shard of the batch, with the exchange carried by
torch.distributed over gloo (parallel.init_data_parallel_host). Both ranks
run on the same GPU; the all-reduce is host-staged, so no kernel waits on
another rank's kernel.

    python tests/dp_worker.py RANK WORLD PORT OUT.npz PRECISION
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def shard_of(n_rows, width, rank, world):
    """Rank's rows of the image (a contiguous band): different ranks touch different voxels."""
    import paper_2205_07058_b200.parallel as par

    r0, rows = par.row_band(n_rows, rank, world)
    return slice(r0 * width, (r0 + rows) * width)


def scene(W=64, res=32):
    import paper_2205_07058_b200.synthetic as S

    sc = S.make_random_scene(7, 4)
    cams = S.hemisphere_cameras(3, 1.8, 7, W, W, 1.5 * W)
    pts = S.occupancy_points(sc, cams, W, W)
    rgb, depth, mask = S.render_gt(sc, cams[0], W, W)
    rays = S.camera_rays(cams[0], W, W)
    return pts, res, W, rays, rgb.reshape(-1, 3), depth.astype(np.float64), (mask > 0.5).astype(np.uint8)


def main():
    rank, world, port, out, precision = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = port
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2205_07058_b200 as P
    from paper_2205_07058_b200.parallel import init_data_parallel_host

    pts, res, W, rays, cgt, depth, alpha = scene()
    ctx = P.Context(0)
    ctx.set_train_precision(precision)
    assert init_data_parallel_host(ctx)
    tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=1), ctx)
    sl = shard_of(W, W, rank, world)
    args = (rays[sl], cgt[sl], depth[sl], alpha[sl])
    res_ = {}
    # gradients of one exchanged step (no update)
    model = P.Model(tree, seed=0, ctx=ctx)
    st = P.LossStats()
    res_["grad_loss"] = P.loss_grads(model, *args, mode="volumetric", stats=st)
    res_["grad_stats"] = np.array([st.rays, st.skipped_rays, st.eta_skipped])
    for k, g in zip(("g_ft", "g_fc", "g_mt", "g_mc"), model.get_grads()):
        res_[k] = g
    # two optimizer steps (surface stage with its pre-surface hits, then volumetric)
    model = P.Model(tree, seed=0, ctx=ctx)
    losses = [P.train_step(model, *args, mode="surface", lr=1e-3),
              P.train_step(model, *args, mode="volumetric", lr=1e-3)]
    res_["losses"] = np.array(losses)
    for k, p in zip(("p_ft", "p_fc", "p_mt", "p_mc"), model.get_params()):
        res_[k] = p
    res_["steps"] = model.get_adam()[2]
    np.savez(out, **res_)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
