"""Regenerate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference built into oracle/_ref):
    python tests/golden/make_golden.py
Every fixture is produced by the reference library itself (ref_shim.cpp over
/root/reference/proj/src); bit-exact geometry comes from the build with
-ffp-contract=off (libsvlf_ref_nofma.so), the default-flag build is recorded
alongside where the two differ. tests/test_golden.py checks the C
restatement (oracle/svlf_oracle.c) and the GPU path against these files.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Reference  # noqa: E402
import paper_2205_07058_b200.synthetic as S  # noqa: E402


def main():
    rn = Reference(nofma=True)
    rf = Reference(nofma=False)

    # 1. octree build (C1: random occupancy res 64, density 0.02, seed 7, dilation 0)
    pts, res, dil, cam, W, H = S.c1_workload()
    t = rn.tree_build(pts, res, dil)
    np.savez_compressed(os.path.join(HERE, "octree_c1.npz"), leaf_codes=t.leaf_codes, corner_ids=t.corner_ids,
                        vertex_count=np.array(t.vertex_count),
                        level_sizes=np.array([len(t.level_codes(l)) for l in range(t.leaf_level + 1)]))

    # 2. traversal: reference test set (16^3, density 0.1, seed 7; random_ray x 200 from Rng(11))
    pts16 = S.random_occupancy_points(16, 0.1, 7)
    t16 = rn.tree_build(pts16, 16, 0)
    rays = S.random_rays(11, 200)
    off, ids, tin, tout = rn.traverse(t16, rays)
    offf, idsf, tinf, toutf = rf.traverse(rf.tree_build(pts16, 16, 0), rays)
    np.savez_compressed(os.path.join(HERE, "traverse_rand16.npz"), rays=rays, offsets=off, ids=ids, t_in=tin,
                        t_out=tout, ids_fma=idsf, t_in_fma=tinf, t_out_fma=toutf)

    # 3. render: C1 scene, 64x64 view, init_model(tree, 1)
    cam64 = S.lookat_camera(tuple(0.5 + 1.8 * c for c in S.C1_EYE_DIR), (0.5, 0.5, 0.5), 64, 64, 96.0)
    m = rn.init_model(t, 1)
    rgb, a, d, st = rn.render_frame(t, m, cam64, 64, 64)
    rgbf, af, df, _ = rf.render_frame(rf.tree_build(pts, res, dil), m, cam64, 64, 64)
    np.savez_compressed(os.path.join(HERE, "render_c1_64.npz"), camera=cam64, rgb=rgb, alpha=a, depth=d, stats=st,
                        rgb_fma=rgbf, alpha_fma=af, depth_fma=df,
                        init_ft_head=m.ft[:256], init_mt_head=m.mt[:256], init_mc_tail=m.mc[-256:])

    # 4. losses + gradients: 24x24 frame of make_random_scene(7, 4), octree res 16 from 2 views
    sc = S.make_random_scene(7, 4)
    cams = S.hemisphere_cameras(2, 1.8, 7, 24, 24, 36.0)
    opts = S.occupancy_points(sc, cams, 24, 24)
    tl = rn.tree_build(opts, 16, 1)
    gt_rgb, gt_d, gt_m = S.render_gt(sc, cams[0], 24, 24)
    lrays = S.camera_rays(cams[0], 24, 24)
    ml = rn.init_model(tl, 0)
    out = {"rays": lrays, "c_gt": gt_rgb, "depth": gt_d.astype(np.float64), "alpha": (gt_m > 0.5).astype(np.uint8),
           "occ_points": opts}
    rng = np.random.default_rng(0)
    for tag, mode, frozen, lw in (("surf", 0, False, (1.0, 0.01, 0.01, 0.1)), ("surf0", 0, False, (1.0, 0.01, 0.0, 0.1)),
                                  ("vol", 1, False, (1.0, 0.01, 0.01, 0.1)), ("volfz", 1, True, (1.0, 0.01, 0.01, 0.1))):
        loss, g, st = rn.loss(tl, ml, lrays, gt_rgb, out["depth"], out["alpha"], mode, lw=lw, frozen=frozen)
        out[f"{tag}_loss"] = np.array(loss)
        out[f"{tag}_stats"] = st
        for k in ("ft", "fc", "mt", "mc"):
            arr = getattr(g, k)
            idx = rng.choice(arr.size, size=64, replace=False)
            out[f"{tag}_{k}_norm"] = np.array(np.linalg.norm(arr.astype(np.float64)))
            out[f"{tag}_{k}_idx"] = idx
            out[f"{tag}_{k}_val"] = arr[idx]
    np.savez_compressed(os.path.join(HERE, "loss_small.npz"), **out)

    # 5. Adam (two steps on fixed vectors)
    p = rng.standard_normal(1000).astype(np.float32)
    g1 = (rng.standard_normal(1000) * 1e-3).astype(np.float32)
    g2 = (rng.standard_normal(1000) * 1e-3).astype(np.float32)
    pm, mm, vm = p.copy(), np.zeros(1000, np.float32), np.zeros(1000, np.float32)
    rn.adam_step(pm, g1, mm, vm, 0, np.float32(1e-3))
    rn.adam_step(pm, g2, mm, vm, 1, np.float32(1e-3))
    np.savez_compressed(os.path.join(HERE, "adam.npz"), p0=p, g1=g1, g2=g2, p=pm, m=mm, v=vm)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
