# Attribution of the render e2e gap (pipelined submit/wait vs the device-timed frame) on C2.
import os
import statistics
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S

ctx = P.Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=4, n_views=100, view_res=400, res=256, dilation=1,
                                               width=1600, ctx=ctx)
tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
model = P.Model(tree, seed=0, ctx=ctx)
camera = P.Camera.from_record(cam, W, H)
n = W * H
flush = torch.empty(160 << 20, dtype=torch.uint8, device="cuda")
prec = "fp16"
d = [torch.empty(k, dtype=torch.float32, device="cuda") for k in (3 * n, n, n)]


def device_loop(k=20, do_flush=True):
    ts = []
    for _ in range(k):
        with torch.cuda.stream(stream):
            if do_flush:
                flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        P.render_frame_device(model, camera, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), precision=prec)
        b.record(stream)
        stream.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


frames = [P.pinned_frame(W, H), P.pinned_frame(W, H)]


def pipe_loop(k=20, do_flush=True):
    P.render_frame_submit(model, camera, frames[0], precision=prec).wait()
    torch.cuda.synchronize()
    sub, wt = [], []
    t0 = time.perf_counter()
    pending = None
    for i in range(k):
        if do_flush:
            with torch.cuda.stream(stream):
                flush.zero_()
        t1 = time.perf_counter()
        tk = P.render_frame_submit(model, camera, frames[i % 2], precision=prec)
        t2 = time.perf_counter()
        if pending is not None:
            pending.wait()
        t3 = time.perf_counter()
        sub.append((t2 - t1) * 1e3)
        wt.append((t3 - t2) * 1e3)
        pending = tk
    pending.wait()
    return (time.perf_counter() - t0) * 1e3 / k, statistics.median(sub), statistics.median(wt)


for _ in range(2):
    print("device loop flush   ms", round(device_loop(), 4), flush=True)
    print("device loop noflush ms", round(device_loop(do_flush=False), 4), flush=True)
    print("pipe flush   ms/frame, submit ms, wait ms", [round(x, 4) for x in pipe_loop()], flush=True)
    print("pipe noflush ms/frame, submit ms, wait ms", [round(x, 4) for x in pipe_loop(do_flush=False)], flush=True)
    os.environ["X"] = "1"
print(ctx.last_timings())
