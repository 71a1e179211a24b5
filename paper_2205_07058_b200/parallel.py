"""Multi-GPU plumbing for the SVLF path.

* Render shards with no collective: the octree and model are replicated and
  each rank renders its own frames / views (weak scaling; a view batch split
  round-robin), or its tiles of one frame (`render_tiles_device`: raster tiles
  dealt round-robin, so clustered foreground spreads over the ranks; or a
  contiguous `row_band`), written into its own buffers.
* Training is data-parallel: the ray batch is split across ranks
  (`shard_slice`); each rank's train step computes loss and gradients of its
  shard, and the library all-reduces them over NCCL (decoders densely,
  feature rows sparsely: union of touched rows) before the replicated Adam
  step. Because the reference's gradients are sums over rays (no 1/N,
  src/train.cpp:473-478), the sum of the shards' gradients is the full
  batch's gradient; any partition is valid.

torch.distributed is used only to rendezvous (share the NCCL id, barriers and
max-over-ranks timing); the gradient traffic goes over the library's own
NCCL communicator.
"""
from __future__ import annotations


def shard_slice(n: int, rank: int, world: int) -> slice:
    """Contiguous, balanced split of n items: rank r gets [r*n//w, (r+1)*n//w)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return slice(rank * n // world, (rank + 1) * n // world)


def row_band(height: int, rank: int, world: int) -> tuple[int, int]:
    """(row0, rows) of rank's band of an image, balanced to within one row."""
    s = shard_slice(height, rank, world)
    return s.start, s.stop - s.start


def tile_origins(width: int, height: int, tile_w: int, tile_h: int, rank: int, world: int):
    """(x0, y0) of the tiles rank owns in a tile-interleaved split of a frame, in the order
    render_tiles_device writes them: raster tile numbers rank, rank + world, ..."""
    tx = width // tile_w
    total = tx * (height // tile_h)
    return [((t % tx) * tile_w, (t // tx) * tile_h) for t in range(rank, total, world)]


def stitch_tiles(image, tiles, width: int, height: int, tile_w: int, tile_h: int, rank: int, world: int):
    """Write rank's tiles (array of k*tile_h*tile_w pixels, any trailing channel dims) into
    `image` (height x width x ...)."""
    t = tiles.reshape(-1, tile_h, tile_w, *image.shape[2:])
    for k, (x0, y0) in enumerate(tile_origins(width, height, tile_w, tile_h, rank, world)):
        image[y0:y0 + tile_h, x0:x0 + tile_w] = t[k]
    return image


def init_data_parallel(ctx, dist=None) -> bool:
    """Attach an NCCL communicator to `ctx` spanning the current
    torch.distributed world (rank 0 creates the id and broadcasts it).
    Returns False (nothing attached) when torch.distributed is not
    initialised."""
    import paper_2205_07058_b200 as P

    if dist is None:
        import torch.distributed as dist
    if not dist.is_initialized():
        return False
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.attach_nccl(obj[0], rank, world)
    return True


def init_data_parallel_host(ctx, dist=None, group=None) -> bool:
    """Attach a host-staged all-reduce (torch.distributed, e.g. the gloo
    backend) to `ctx` instead of NCCL: the library stages each exchange buffer
    in page-locked host memory and this callback reduces it in place. Same
    exchange, same results; used where NCCL peers are unavailable (CPU-side
    frameworks, tests with several ranks on one GPU). Returns False when
    torch.distributed is not initialised."""
    import numpy as np
    import torch

    if dist is None:
        import torch.distributed as dist
    if not dist.is_initialized():
        return False
    ops = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX}

    def allreduce(buf: np.ndarray, op: str):
        t = torch.from_numpy(buf)  # shares the staging memory
        if buf.dtype == np.uint8:  # gloo has no uint8 max: reduce a wider copy
            w = t.to(torch.int32)
            dist.all_reduce(w, op=ops[op], group=group)
            t.copy_(w.to(torch.uint8))
        else:
            dist.all_reduce(t, op=ops[op], group=group)

    ctx.attach_host_collective(allreduce, dist.get_rank(group), dist.get_world_size(group))
    return True
