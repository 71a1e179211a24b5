# Host-link probe for the train e2e leg: raw pinned H2D bandwidth, and C3 train_step with
# pageable vs page-locked host batches (and the staged/pipelined API when present).
import os
import statistics
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S

x = torch.empty(18 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(18 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print(f"pinned H2D 18 MiB: {18 * 20 / 1024 / (time.perf_counter() - t0):.2f} GB/s", flush=True)

sc, cam, pts, res, dil, rays, cgt, depth, alpha = S.c3_workload()
ctx = P.Context(0)
tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
model = P.Model(tree, seed=0, ctx=ctx)
cgt = np.ascontiguousarray(cgt, dtype=np.float32)
alpha = np.ascontiguousarray(alpha, dtype=np.uint8)


def pin(a):
    p = P.pinned_empty(a.size, a.dtype)
    p[:] = a.reshape(-1)
    return p.reshape(a.shape)


pinned = [pin(np.ascontiguousarray(a)) for a in (rays, cgt, depth, alpha)]


def timed(fn, k=10):
    for _ in range(3):
        fn()
    t = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        t.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(t)


print("pageable train_step ms", timed(lambda: P.train_step(model, rays, cgt, depth, alpha, lr=2e-4)), flush=True)
print("pinned   train_step ms", timed(lambda: P.train_step(model, *pinned, lr=2e-4)), flush=True)
print("timings", ctx.last_timings(), flush=True)
if hasattr(P, "TrainPipeline"):
    for src, name in ((pinned, "pinned"), ((rays, cgt, depth, alpha), "pageable")):
        pipe = P.TrainPipeline(model)
        k = 20
        pipe.stage(*src)
        for _ in range(3):
            pipe.stage(*src)
            pipe.step(lr=2e-4)
        t0 = time.perf_counter()
        for _ in range(k):
            pipe.stage(*src)
            pipe.step(lr=2e-4)
        ms = (time.perf_counter() - t0) * 1e3 / k
        pipe.drain()
        print(f"pipelined {name} ms/step {ms:.3f} -> {rays.shape[0] / ms / 1e3:.1f} Mrays/s", flush=True)
