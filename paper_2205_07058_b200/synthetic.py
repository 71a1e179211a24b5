"""Synthetic inputs for the benchmarks and examples.

Restates the reference's input generators so workloads are the reference's
own scenes, bit for bit:
  * Rng: splitmix64-seeded MT19937-64 with the 53-bit uniform mapping and
    named sub-streams (include/svlf/rng.hpp:9-50);
  * make_random_scene (src/scene.cpp:92-124), sample_hemisphere_cameras
    (src/scene.cpp:126-141), make_lookat_camera (src/camera.cpp:24-40);
  * raycast + shade (src/scene.cpp:56-90) vectorised with numpy (IEEE
    +,-,*,/,sqrt only, so per-pixel results equal the scalar C++);
  * occupancy points by back-projecting foreground depth exactly as train()
    does (ray.at(float depth), src/train.cpp:376-386);
  * random_occupancy / random_ray from tests/test_octree.cpp:38-64.
This is input generation only (reference scope "OUT OF SCOPE: synthetic-input
generator"); it is not on the measured path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_M64 = (1 << 64) - 1


def _mix64(x):
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


class Rng:
    """include/svlf/rng.hpp: MT19937-64 seeded with mix64(seed)."""

    def __init__(self, seed: int):
        self.seed = seed & _M64
        mt = [0] * 312
        mt[0] = _mix64(self.seed)
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self._mt = mt
        self._i = 312

    def _twist(self):
        mt = self._mt
        UM, LM, A = 0xFFFFFFFF80000000, 0x7FFFFFFF, 0xB5026F5AA96619E9
        for i in range(312):
            x = (mt[i] & UM) | (mt[(i + 1) % 312] & LM)
            xa = x >> 1
            if x & 1:
                xa ^= A
            mt[i] = mt[(i + 156) % 312] ^ xa
        self._i = 0

    def next_u64(self) -> int:
        if self._i >= 312:
            self._twist()
        x = self._mt[self._i]
        self._i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = float(self.next_u64() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def below(self, n: int) -> int:
        return self.next_u64() % n

    def sub(self, stream: int) -> "Rng":
        return Rng(self.seed ^ _mix64((stream + 0x51ED2700) & _M64))


STREAM_SCENE = 6
STREAM_CAMERAS = 7


# ---- vector helpers (IEEE double, reference operand order) -----------------
def _norm(v):
    return math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])


def _normalized(v):
    n = _norm(v)
    return (v[0] / n, v[1] / n, v[2] / n)


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def lookat_camera(eye, target, width, height, focal):
    """make_lookat_camera (src/camera.cpp:24-40) -> record (fx, fy, cx, cy, c2w[16])."""
    f = _normalized((target[0] - eye[0], target[1] - eye[1], target[2] - eye[2]))
    up = (0.0, 0.0, 1.0)
    if abs(f[0] * up[0] + f[1] * up[1] + f[2] * up[2]) > 0.999:
        up = (0.0, 1.0, 0.0)
    right = _normalized(_cross(f, up))
    down = _cross(f, right)
    c2w = [right[0], down[0], f[0], eye[0], right[1], down[1], f[1], eye[1],
           right[2], down[2], f[2], eye[2], 0.0, 0.0, 0.0, 1.0]
    return np.array([focal, focal, width * 0.5, height * 0.5] + c2w, dtype=np.float64)


def hemisphere_cameras(n, radius, seed, width, height, focal):
    """sample_hemisphere_cameras (src/scene.cpp:126-141) -> n x 20 records."""
    rng = Rng(seed).sub(STREAM_CAMERAS)
    out = []
    for _ in range(n):
        z = rng.uniform()
        az = rng.uniform(0.0, 2.0 * math.pi)
        r = math.sqrt(max(0.0, 1.0 - z * z))
        d = (r * math.cos(az), r * math.sin(az), z)
        eye = (0.5 + d[0] * radius, 0.5 + d[1] * radius, 0.5 + d[2] * radius)
        out.append(lookat_camera(eye, (0.5, 0.5, 0.5), width, height, focal))
    return np.stack(out)


@dataclass
class Scene:
    spheres: list = field(default_factory=list)  # (center(3), radius, albedo(3))
    boxes: list = field(default_factory=list)    # (lo(3), hi(3), albedo(3))
    light_dir: tuple = (0.0, 0.0, -1.0)
    light_rgb: tuple = (0.7, 0.7, 0.7)
    ambient: tuple = (0.25, 0.25, 0.25)
    background: tuple = (0.0, 0.0, 0.0)


def make_random_scene(seed, n_primitives):
    """make_random_scene (src/scene.cpp:92-124)."""
    rng = Rng(seed).sub(STREAM_SCENE)
    sc = Scene()
    for _ in range(n_primitives):
        albedo = (rng.uniform(0.2, 1.0), rng.uniform(0.2, 1.0), rng.uniform(0.2, 1.0))
        if rng.uniform() < 0.5:
            radius = rng.uniform(0.08, 0.16)
            c = (rng.uniform(0.25, 0.75), rng.uniform(0.25, 0.75), rng.uniform(0.25, 0.75))
            sc.spheres.append((c, radius, albedo))
        else:
            half = (rng.uniform(0.05, 0.12), rng.uniform(0.05, 0.12), rng.uniform(0.05, 0.12))
            c = (rng.uniform(0.25, 0.75), rng.uniform(0.25, 0.75), rng.uniform(0.25, 0.75))
            lo = (c[0] - half[0], c[1] - half[1], c[2] - half[2])
            hi = (c[0] + half[0], c[1] + half[1], c[2] + half[2])
            sc.boxes.append((lo, hi, albedo))
    az = rng.uniform(0.0, 2.0 * math.pi)
    el = rng.uniform(0.35, 1.2)
    ld = _normalized((math.cos(az) * math.cos(el), math.sin(az) * math.cos(el), math.sin(el)))
    sc.light_dir = (-ld[0], -ld[1], -ld[2])
    return sc


def camera_rays(cam, width, height):
    """Camera::pixel_ray for every pixel in raster order -> (W*H) x 6."""
    cam = np.asarray(cam, dtype=np.float64)
    fx, fy, cx, cy = cam[:4]
    m = cam[4:20]
    px = np.arange(width * height, dtype=np.int64)
    ix = (px % width).astype(np.float64)
    iy = (px // width).astype(np.float64)
    vx = ((ix + 0.5) - cx) / fx
    vy = ((iy + 0.5) - cy) / fy
    vz = 1.0
    r = [(m[4 * i] * vx + m[4 * i + 1] * vy) + m[4 * i + 2] * vz for i in range(3)]
    n = np.sqrt((r[0] * r[0] + r[1] * r[1]) + r[2] * r[2])
    out = np.empty((width * height, 6))
    out[:, 0], out[:, 1], out[:, 2] = m[3], m[7], m[11]
    out[:, 3], out[:, 4], out[:, 5] = r[0] / n, r[1] / n, r[2] / n
    return out


def _ray_aabb(o, d, lo, hi):
    """Vectorised src/geometry.cpp:5-26 -> (hit mask, t0, t1)."""
    n = o.shape[0]
    t0 = np.zeros(n)
    t1 = np.full(n, np.inf)
    ok = np.ones(n, dtype=bool)
    for a in range(3):
        da, oa = d[:, a], o[:, a]
        zero = da == 0.0
        ok &= ~(zero & ((oa < lo[a]) | (oa > hi[a])))
        with np.errstate(divide="ignore", invalid="ignore"):
            inv = 1.0 / np.where(zero, 1.0, da)
            ta = (lo[a] - oa) * inv
            tb = (hi[a] - oa) * inv
        lo_t = np.minimum(ta, tb)
        hi_t = np.maximum(ta, tb)
        upd0 = ~zero & (lo_t > t0)
        t0 = np.where(upd0, lo_t, t0)
        upd1 = ~zero & (hi_t < t1)
        t1 = np.where(upd1, hi_t, t1)
        ok &= ~(t1 < t0)
    return ok, t0, t1


def _raycast(sc: Scene, o, d):
    """raycast (src/scene.cpp:56-77) vectorised -> (hit, t, point, normal, albedo)."""
    n = o.shape[0]
    eps = 1e-9
    best_t = np.full(n, np.inf)
    have = np.zeros(n, dtype=bool)
    normal = np.zeros((n, 3))
    albedo = np.zeros((n, 3))
    point = np.zeros((n, 3))
    for c, r, alb in sc.spheres:
        oc = o - np.asarray(c)
        b = (oc[:, 0] * d[:, 0] + oc[:, 1] * d[:, 1]) + oc[:, 2] * d[:, 2]
        cc = ((oc[:, 0] * oc[:, 0] + oc[:, 1] * oc[:, 1]) + oc[:, 2] * oc[:, 2]) - r * r
        disc = b * b - cc
        valid = disc >= 0
        sq = np.sqrt(np.where(valid, disc, 0.0))
        ta = -b - sq
        tb = -b + sq
        t = np.where(ta > eps, ta, np.where(tb > eps, tb, np.nan))
        valid &= ~np.isnan(t)
        upd = valid & (~have | (t < best_t))
        if upd.any():
            p = o[upd] + d[upd] * t[upd, None]
            v = p - np.asarray(c)
            nn = np.sqrt((v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2])
            best_t[upd] = t[upd]
            point[upd] = p
            normal[upd] = v / nn[:, None]
            albedo[upd] = alb
            have |= upd
    for lo, hi, alb in sc.boxes:
        ok, t0, t1 = _ray_aabb(o, d, lo, hi)
        t = np.where(t0 > eps, t0, np.where(t1 > eps, t1, -1.0))
        upd = ok & (t > 0) & (~have | (t < best_t))
        if upd.any():
            p = o[upd] + d[upd] * t[upd, None]
            dd = np.stack([p[:, 0] - lo[0], hi[0] - p[:, 0], p[:, 1] - lo[1], hi[1] - p[:, 1],
                           p[:, 2] - lo[2], hi[2] - p[:, 2]], axis=1)
            best = np.argmin(dd, axis=1)  # first minimum, as the reference's strict '<' scan
            table = np.array([[-1, 0, 0], [1, 0, 0], [0, -1, 0], [0, 1, 0], [0, 0, -1], [0, 0, 1]], float)
            best_t[upd] = t[upd]
            point[upd] = p
            normal[upd] = table[best]
            albedo[upd] = alb
            have |= upd
    return have, best_t, point, normal, albedo


def render_gt(sc: Scene, cam, width, height):
    """generate_dataset's pixel loop (src/dataset.cpp:61-83): rgb, depth, mask (float32)."""
    rays = camera_rays(cam, width, height)
    o, d = rays[:, :3], rays[:, 3:]
    have, t, p, nrm, alb = _raycast(sc, o, d)
    nl = -np.asarray(sc.light_dir)
    direct = np.maximum(0.0, (nrm[:, 0] * nl[0] + nrm[:, 1] * nl[1]) + nrm[:, 2] * nl[2])
    lit = have & (direct > 0)
    if lit.any():
        so = p[lit] + nrm[lit] * 1e-6
        sd = np.broadcast_to(nl, so.shape).copy()
        blocked, *_ = _raycast(sc, so, sd)
        idx = np.nonzero(lit)[0]
        direct[idx[blocked]] = 0.0
    amb = np.asarray(sc.ambient)
    lrgb = np.asarray(sc.light_rgb)
    col = alb * (amb[None, :] + lrgb[None, :] * direct[:, None])
    col = np.clip(col, 0.0, 1.0)
    rgb = np.where(have[:, None], col, np.asarray(sc.background)[None, :]).astype(np.float32)
    depth = np.where(have, t, 0.0).astype(np.float32)
    mask = have.astype(np.float32)
    return rgb.reshape(-1), depth, mask


def backproject(cam, width, height, depth):
    """Foreground depth -> world points, ray.at(double(float depth)) (src/train.cpp:376-386)."""
    rays = camera_rays(cam, width, height)
    fg = depth > 0.0
    d = depth[fg].astype(np.float64)
    return rays[fg, :3] + rays[fg, 3:] * d[:, None]


def occupancy_points(scene, cams, width, height):
    pts = []
    for c in cams:
        _, depth, _ = render_gt(scene, c, width, height)
        pts.append(backproject(c, width, height, depth))
    return np.concatenate(pts)


def random_occupancy_points(res, density, seed):
    """tests/test_octree.cpp:38-48 (cell centres kept with probability `density`)."""
    rng = Rng(seed)
    h = 1.0 / res
    pts = []
    for z in range(res):
        for y in range(res):
            for x in range(res):
                if rng.uniform() < density:
                    pts.append(((x + 0.5) * h, (y + 0.5) * h, (z + 0.5) * h))
    return np.array(pts, dtype=np.float64)


def random_rays(seed, n):
    """tests/test_octree.cpp:50-64 random_ray() x n from one Rng(seed)."""
    rng = Rng(seed)
    out = np.zeros((n, 6))
    for i in range(n):
        if rng.uniform() < 0.5:
            az = rng.uniform(0, 2 * math.pi)
            el = rng.uniform(-math.pi / 2, math.pi / 2)
            v = (math.cos(az) * math.cos(el), math.sin(az) * math.cos(el), math.sin(el))
            origin = (0.5 + v[0] * 2.0, 0.5 + v[1] * 2.0, 0.5 + v[2] * 2.0)
        else:
            origin = (rng.uniform(), rng.uniform(), rng.uniform())
        target = [rng.uniform(), rng.uniform(), rng.uniform()]
        if _norm((target[0] - origin[0], target[1] - origin[1], target[2] - origin[2])) < 1e-9:
            target[0] += 0.1
        d = _normalized((target[0] - origin[0], target[1] - origin[1], target[2] - origin[2]))
        out[i] = (*origin, *d)
    return out


# ---- benchmark workloads (BASELINE.json configs) -----------------------------
C1_EYE_DIR = (0.6, 0.3, 0.7416)


def c1_workload():
    """Config 1: random occupancy res 64, density 0.02, seed 7, dilation 0; 200x200 view."""
    pts = random_occupancy_points(64, 0.02, 7)
    eye = tuple(0.5 + 1.8 * c for c in C1_EYE_DIR)
    cam = lookat_camera(eye, (0.5, 0.5, 0.5), 200, 200, 300.0)
    return pts, 64, 0, cam, 200, 200


def occupancy_points_gpu(ctx, sc: Scene, cams, width, height):
    """occupancy_points via the GPU ground truth + back-projection (bit-identical
    depth and points; order differs, which the octree build ignores) -> numpy."""
    import torch

    import paper_2205_07058_b200 as P

    n = width * height
    dev = torch.device("cuda", ctx.device)
    rgb = torch.empty(3 * n, dtype=torch.float32, device=dev)
    depth = torch.empty(n, dtype=torch.float32, device=dev)
    mask = torch.empty(n, dtype=torch.float32, device=dev)
    pts = torch.empty((len(cams) * n, 3), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    total = 0
    for c in cams:
        cam = P.Camera.from_record(c, width, height)
        P.render_gt_device(ctx, sc, cam, rgb.data_ptr(), depth.data_ptr(), mask.data_ptr())
        total += P.backproject_device(ctx, cam, depth.data_ptr(), pts.data_ptr() + total * 24, n)
    return pts[:total].cpu().numpy()


def rtmv_workload(n_objects=4, n_views=100, view_res=400, res=256, dilation=1, width=1600, seed=7, ctx=None):
    """Config 2: RTMV-shaped scene (make_random_scene(7, n)), occupancy from
    n_views hemisphere depth maps at view_res^2, octree res 256 (depth 8),
    render width^2 at focal 1.5*width from the survey's eye direction.
    With a context the ground truth and back-projection run on the GPU."""
    sc = make_random_scene(seed, n_objects)
    cams = hemisphere_cameras(n_views, 1.8, seed, view_res, view_res, 1.5 * view_res)
    pts = (occupancy_points_gpu(ctx, sc, cams, view_res, view_res) if ctx is not None
           else occupancy_points(sc, cams, view_res, view_res))
    eye = tuple(0.5 + 1.8 * c for c in C1_EYE_DIR)
    cam = lookat_camera(eye, (0.5, 0.5, 0.5), width, width, 1.5 * width)
    return sc, pts, res, dilation, cam, width, width


def c3_workload(width=512, objects=4, res=256, dilation=1, seed=7):
    """Config 3: one hemisphere frame (width^2 rays, 2^18 at 512) of make_random_scene(seed, objects)
    with ground truth from the analytic ray-caster; the octree is train()'s occupancy for that
    one-frame dataset (back-projected foreground depth, res 256 = depth 8, dilation 1)."""
    sc = make_random_scene(seed, objects)
    cam = hemisphere_cameras(1, 1.8, seed, width, width, 1.5 * width)[0]
    rgb, depth, mask = render_gt(sc, cam, width, width)
    pts = backproject(cam, width, width, depth)
    rays = camera_rays(cam, width, width)
    return sc, cam, pts, res, dilation, rays, rgb.reshape(-1, 3), depth.astype(np.float64), (mask > 0.5)


def render_gt_gpu(ctx, sc: Scene, cam, width, height):
    """render_gt on the GPU (svlf_render_gt_device) -> numpy (rgb, depth, mask)."""
    import torch

    import paper_2205_07058_b200 as P

    n = width * height
    dev = torch.device("cuda", ctx.device)
    rgb = torch.empty(3 * n, dtype=torch.float32, device=dev)
    depth = torch.empty(n, dtype=torch.float32, device=dev)
    mask = torch.empty(n, dtype=torch.float32, device=dev)
    torch.cuda.synchronize(dev)
    P.render_gt_device(ctx, sc, P.Camera.from_record(cam, width, height), rgb.data_ptr(), depth.data_ptr(),
                       mask.data_ptr())
    return rgb.cpu().numpy(), depth.cpu().numpy(), mask.cpu().numpy()


def occupancy_octree_gpu(ctx, sc: Scene, cams, width, height, grid):
    """train()'s occupancy pipeline entirely on the GPU: ground-truth depth per view,
    back-projection of the foreground, octree build from the device-resident points."""
    import torch

    import paper_2205_07058_b200 as P

    n = width * height
    dev = torch.device("cuda", ctx.device)
    rgb = torch.empty(3 * n, dtype=torch.float32, device=dev)
    depth = torch.empty(n, dtype=torch.float32, device=dev)
    mask = torch.empty(n, dtype=torch.float32, device=dev)
    pts = torch.empty((len(cams) * n, 3), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    total = 0
    for c in cams:
        cam = P.Camera.from_record(c, width, height)
        P.render_gt_device(ctx, sc, cam, rgb.data_ptr(), depth.data_ptr(), mask.data_ptr())
        total += P.backproject_device(ctx, cam, depth.data_ptr(), pts.data_ptr() + total * 24, n)
    return P.SparseOctree.build_device(pts.data_ptr(), total, grid, ctx), total
