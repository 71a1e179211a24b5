# f_C chain phase latencies (clock64 per phase, chains of CTA 0): run with SVLF_LIB_PATH pointing at a
# build made with -DSVLF_DEC_TRACE=1 (make -C paper_2205_07058_b200/csrc OUT=... SVLF_DEFS=-DSVLF_DEC_TRACE=1).
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2205_07058_b200 as P
import paper_2205_07058_b200.synthetic as S
ctx = P.Context(0)
sc, pts, res, dil, cam, W, H = S.rtmv_workload(n_objects=4, n_views=100, view_res=400, res=256, dilation=1, width=1600, ctx=ctx)
tree = P.SparseOctree.build(pts, P.GridConfig(res, dilation=dil), ctx)
model = P.Model(tree, seed=0, ctx=ctx)
camera = P.Camera.from_record(cam, W, H)
n = W * H
d = [torch.empty(k, dtype=torch.float32, device="cuda") for k in (3 * n, n, n)]
for _ in range(4):
    P.render_frame_device(model, camera, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), precision="fp16")
torch.cuda.synchronize()
L = C.CDLL(os.environ["SVLF_LIB_PATH"])
buf = np.zeros((3, 64, 10), np.uint64)
if hasattr(L, "svlf_debug_dec_trace"):
    assert L.svlf_debug_dec_trace(buf.ctypes.data_as(C.c_void_p)) == 0
names = ["wait_full", "L0", "epi0", "L1", "epi1", "L2", "epi2", "head", "out", "next"]
for ch in range(3):
    b = buf[ch].astype(np.int64)
    ok = b[:, 0] > 0
    b = b[ok]
    if len(b) < 4: continue
    dd = np.diff(b, axis=1)
    nxt = b[1:, 0] - b[:-1, 9]
    print(f"chain {ch}: tiles {len(b)} per-tile cycles median {np.median(b[1:,0]-b[:-1,0]):.0f}")
    for i in range(9):
        print(f"   {names[i]:10s} {np.median(dd[2:, i]):8.0f}")
    print(f"   {'next':10s} {np.median(nxt[2:]):8.0f}")
ts = []
for _ in range(10):
    P.render_frame_device(model, camera, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), precision="fp16")
    ts.append(ctx.last_timings()["decode_ms"])
print("decode_ms", round(float(np.median(ts)), 4))
