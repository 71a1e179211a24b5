# Runs a few C3 train steps through train_step_device (used by profiles/run_profiles.sh under ncu).
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S
sc, cam, pts, res, dil, rays, cgt, depth, alpha = S.c3_workload()
ctx = P.Context(0)
if len(sys.argv) > 3:
    ctx.set_train_precision(sys.argv[3])
tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
model = P.Model(tree, seed=0, ctx=ctx)
n = rays.shape[0]
d_rays = torch.from_numpy(np.ascontiguousarray(rays)).cuda()
d_cgt = torch.from_numpy(np.ascontiguousarray(cgt, dtype=np.float32)).cuda()
d_depth = torch.from_numpy(np.ascontiguousarray(depth)).cuda()
d_alpha = torch.from_numpy(np.ascontiguousarray(alpha, dtype=np.uint8)).cuda()
mode = sys.argv[1] if len(sys.argv) > 1 else "volumetric"
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    t0 = time.perf_counter()
    loss = P.train_step_device(model, d_rays.data_ptr(), d_cgt.data_ptr(), d_depth.data_ptr(), d_alpha.data_ptr(), n, mode=mode, lr=2e-4)
    torch.cuda.synchronize()
    print(k, loss, (time.perf_counter() - t0) * 1e3, ctx.last_timings())
