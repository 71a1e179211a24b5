"""Data-parallel decomposition on CPU with torch.distributed/gloo, world 2.

Each rank evaluates the oracle's loss and gradients on its shard of the ray
batch (paper_2205_07058_b200.parallel.shard_slice); the shards are summed with
an all-reduce and must equal the full-batch loss/gradients. The reference's
gradients are sums over rays (src/train.cpp:473-478), which is the invariant
the library's NCCL exchange (train.cu, data-parallel block) relies on: dense
sum of decoder gradients + sum over the union of touched feature rows, then
the replicated Adam step. Also checks the shard/row-band helpers."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2205_07058_b200.parallel import row_band, shard_slice

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import paper_2205_07058_b200.synthetic as S
    from oracle import Oracle

    W = 24
    sc = S.make_random_scene(7, 4)
    cams = S.hemisphere_cameras(2, 1.8, 7, W, W, 1.5 * W)
    pts = S.occupancy_points(sc, cams, W, W)
    rgb, depth, mask = S.render_gt(sc, cams[0], W, W)
    o = Oracle()
    t = o.tree_build(pts, 16, 1)
    m = o.init_model(t, 0)
    return o, t, m, S.camera_rays(cams[0], W, W), rgb.reshape(-1, 3), depth.astype(np.float64), \
        (mask > 0.5).astype(np.uint8)


def _flat(g):
    return np.concatenate([g.ft, g.fc, g.mt, g.mc]).astype(np.float64)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    o, t, m, rays, cgt, depth, alpha = _problem()
    sl = shard_slice(rays.shape[0], rank, world)
    loss, g, st = o.loss(t, m, rays[sl], cgt[sl], depth[sl], alpha[sl], 1)
    vec = torch.from_numpy(_flat(g))
    tot = torch.tensor([loss] + [float(x) for x in st], dtype=torch.float64)
    # touched feature rows: the union is what the library exchanges sparsely
    touched = torch.from_numpy((np.abs(g.ft.reshape(-1, 64)).sum(1) > 0).astype(np.uint8))
    dist.all_reduce(vec)
    dist.all_reduce(tot)
    dist.all_reduce(touched, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((vec.numpy(), tot.numpy(), touched.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gradients_sum_to_full_batch():
    pytest.importorskip("torch.distributed")
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    vec, tot, touched = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    o, t, m, rays, cgt, depth, alpha = _problem()
    loss, g, st = o.loss(t, m, rays, cgt, depth, alpha, 1)
    full = _flat(g)
    assert tot[0] == pytest.approx(loss, rel=1e-12)
    assert tot[1:].tolist() == [float(x) for x in st]
    assert np.linalg.norm(vec - full) <= 1e-5 * np.linalg.norm(full)
    # rows outside the union of touched rows carry exactly zero gradient in the full batch
    ft = g.ft.reshape(-1, 64)
    assert not np.any(ft[touched == 0])
    assert touched.sum() > 0


def test_shard_helpers():
    for n in (0, 1, 7, 1600, 2 ** 18):
        for w in (1, 2, 3, 8):
            parts = [shard_slice(n, r, w) for r in range(w)]
            assert parts[0].start == 0 and parts[-1].stop == n
            assert all(a.stop == b.start for a, b in zip(parts, parts[1:]))
            sizes = [p.stop - p.start for p in parts]
            assert max(sizes) - min(sizes) <= 1
    bands = [row_band(1600, r, 8) for r in range(8)]
    assert sum(b[1] for b in bands) == 1600 and bands[3] == (600, 200)
    with pytest.raises(ValueError):
        shard_slice(10, 2, 2)
