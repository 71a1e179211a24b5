"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two checkers share one numpy-level interface:

* ``Oracle``    -- oracle/build/libsvlf_oracle.so, the plain-C restatement of the
                   reference algorithms (oracle/svlf_oracle.c). Always buildable.
* ``Reference`` -- oracle/_ref/libsvlf_ref{,_nofma}.so, the UNMODIFIED reference
                   sources (/root/reference/proj/src) behind oracle/ref/ref_shim.cpp.
                   Present wherever it was built (it travels to the GPU box as a
                   prebuilt file); tests that need it skip when it is absent.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module. The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libsvlf_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsvlf_ref.so")
REF_NOFMA_SO = os.path.join(HERE, "_ref", "libsvlf_ref_nofma.so")

MT_SIZE = 17538
MC_SIZE = 38403
LAYERS_T = (134, 128, 2)
LAYERS_C = (38, 128, 128, 128, 3)

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


def build_oracle() -> None:
    """Compile the C restatement (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def mlp_layout(dims):
    """[(w_off, w_shape, b_off, b_len)] of the flat decoder layout."""
    out, o = [], 0
    for i, o_dim in zip(dims[:-1], dims[1:]):
        out.append((o, (o_dim, i), o + i * o_dim, o_dim))
        o += i * o_dim + o_dim
    return out


class Model:
    """Flat-parameter SVLF model: feature volumes + two decoders (numpy f32)."""

    def __init__(self, ft, fc, mt, mc):
        self.ft = _f32(ft)
        self.fc = _f32(fc)
        self.mt = _f32(mt)
        self.mc = _f32(mc)

    def copy(self):
        return Model(self.ft.copy(), self.fc.copy(), self.mt.copy(), self.mc.copy())

    @property
    def vertex_count(self):
        return self.ft.size // 64


class _TreeBase:
    def level_codes(self, level):  # pragma: no cover - abstract
        raise NotImplementedError


class Oracle:
    """The C restatement."""

    kind = "port"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        L = self.lib = C.CDLL(path)
        L.or_last_error.restype = C.c_char_p
        L.or_tree_build.restype = C.c_void_p
        L.or_tree_build.argtypes = [_dp, C.c_size_t, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
        L.or_tree_from_leaves.restype = C.c_void_p
        L.or_tree_from_leaves.argtypes = [_u64p, C.c_size_t, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
        L.or_tree_free.argtypes = [C.c_void_p]
        L.or_tree_leaf_level.argtypes = [C.c_void_p]
        L.or_tree_level_size.restype = C.c_size_t
        L.or_tree_level_size.argtypes = [C.c_void_p, C.c_int]
        L.or_tree_level_codes.restype = C.POINTER(C.c_uint64)
        L.or_tree_level_codes.argtypes = [C.c_void_p, C.c_int]
        L.or_tree_corner_ids.restype = C.POINTER(C.c_uint32)
        L.or_tree_corner_ids.argtypes = [C.c_void_p]
        L.or_tree_vertex_count.restype = C.c_uint32
        L.or_tree_vertex_count.argtypes = [C.c_void_p]
        L.or_tree_dropped.restype = C.c_size_t
        L.or_tree_dropped.argtypes = [C.c_void_p]
        L.or_tree_locate.argtypes = [C.c_void_p, _dp, C.POINTER(C.c_uint64)]
        L.or_ray_aabb.argtypes = [_dp, _dp, _dp, _dp]
        L.or_traverse.restype = C.c_size_t
        L.or_traverse.argtypes = [C.c_void_p, _dp, C.c_size_t, _u64p, C.c_size_t, _u64p, _dp, _dp]
        L.or_rng_u64_first.restype = C.c_uint64
        L.or_rng_u64_first.argtypes = [C.c_uint64]
        L.or_init_model.argtypes = [C.c_void_p, C.c_uint64, _fp, _fp, _fp, _fp]
        L.or_lookat_camera.argtypes = [_dp, _dp, C.c_uint32, C.c_uint32, C.c_double, _dp]
        L.or_camera_rays.argtypes = [_dp, C.c_uint32, C.c_uint32, _dp]
        L.or_hemisphere_cameras.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, _dp]
        L.or_scene_make.restype = C.c_void_p
        L.or_scene_make.argtypes = [C.c_uint64, C.c_int]
        L.or_scene_free.argtypes = [C.c_void_p]
        L.or_scene_render_gt.argtypes = [C.c_void_p, _dp, C.c_uint32, C.c_uint32, _fp, _fp, _fp]
        L.or_render_rays.argtypes = [C.c_void_p, _fp, _fp, _fp, _fp, _dp, C.c_size_t, C.c_void_p, _fp, _fp, _fp, _i64p]
        L.or_render_frame.argtypes = [C.c_void_p, _fp, _fp, _fp, _fp, _dp, C.c_uint32, C.c_uint32, C.c_void_p, _fp, _fp, _fp, _i64p]
        L.or_loss.argtypes = [C.c_void_p, _fp, _fp, _fp, _fp, _dp, _fp, _dp, _u8p, C.c_size_t, C.c_int, _dp, C.c_int,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _i64p, C.POINTER(C.c_double)]
        L.or_adam_step.argtypes = [_fp, _fp, _fp, _fp, C.c_size_t, C.c_uint64, C.c_float]

    def _err(self):
        return OracleError(self.lib.or_last_error().decode())

    # ---- octree ------------------------------------------------------
    def tree_build(self, points, res, dilation=1, lo=None, hi=None):
        pts = _f64(points).reshape(-1, 3)
        h = self.lib.or_tree_build(pts, pts.shape[0], res, dilation, _box(lo), _box(hi))
        if not h:
            raise self._err()
        return OTree(self, h, res, dilation, lo, hi)

    def tree_from_leaves(self, codes, res, dilation=1, lo=None, hi=None):
        c = np.ascontiguousarray(codes, dtype=np.uint64)
        h = self.lib.or_tree_from_leaves(c, c.size, res, dilation, _box(lo), _box(hi))
        if not h:
            raise self._err()
        return OTree(self, h, res, dilation, lo, hi)

    def ray_aabb(self, ray6, lo, hi):
        t = np.zeros(2)
        ok = self.lib.or_ray_aabb(_f64(ray6), _f64(lo), _f64(hi), t)
        return (t[0], t[1]) if ok else None

    def node_tests(self, reset=True):
        """ray_aabb calls of traverse() on this thread since the last reset (src/octree.cpp:185-235)."""
        self.lib.or_node_tests.restype = C.c_uint64
        self.lib.or_node_tests.argtypes = [C.c_int]
        return int(self.lib.or_node_tests(1 if reset else 0))

    def traverse(self, tree, rays):
        rays = _f64(rays).reshape(-1, 6)
        n = rays.shape[0]
        off = np.zeros(n + 1, dtype=np.uint64)
        e64, ed = np.zeros(1, np.uint64), np.zeros(1)
        total = self.lib.or_traverse(tree.h, rays, n, off, 0, e64, ed, ed)
        ids = np.zeros(max(total, 1), np.uint64)
        tin, tout = np.zeros(max(total, 1)), np.zeros(max(total, 1))
        self.lib.or_traverse(tree.h, rays, n, off, total, ids, tin, tout)
        return off.astype(np.int64), ids[:total], tin[:total], tout[:total]

    # ---- model / cameras / scenes -----------------------------------
    def init_model(self, tree, seed):
        V = tree.vertex_count
        m = Model(np.zeros(V * 64, np.float32), np.zeros(V * 32, np.float32),
                  np.zeros(MT_SIZE, np.float32), np.zeros(MC_SIZE, np.float32))
        self.lib.or_init_model(tree.h, seed, m.ft, m.fc, m.mt, m.mc)
        return m

    def lookat_camera(self, eye, target, w, h, focal):
        out = np.zeros(20)
        self.lib.or_lookat_camera(_f64(eye), _f64(target), w, h, focal, out)
        return out

    def camera_rays(self, cam, w, h):
        out = np.zeros((w * h, 6))
        self.lib.or_camera_rays(_f64(cam), w, h, out)
        return out

    def hemisphere_cameras(self, n, radius, seed, w, h, focal):
        out = np.zeros((n, 20))
        self.lib.or_hemisphere_cameras(n, radius, seed, w, h, focal, out)
        return out

    def scene_make(self, seed, prims):
        return OScene(self, self.lib.or_scene_make(seed, prims))

    def scene_render_gt(self, scene, cam, w, h):
        rgb = np.zeros(w * h * 3, np.float32)
        depth = np.zeros(w * h, np.float32)
        mask = np.zeros(w * h, np.float32)
        self.lib.or_scene_render_gt(scene.h, _f64(cam), w, h, rgb, depth, mask)
        return rgb, depth, mask

    # ---- render / loss ----------------------------------------------
    def render_rays(self, tree, m, rays, bg=None):
        rays = _f64(rays).reshape(-1, 6)
        n = rays.shape[0]
        rgb, a, d = np.zeros(n * 3, np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32)
        st = np.zeros(5, np.int64)
        bgp = _f32(bg).ctypes.data if bg is not None else None
        if self.lib.or_render_rays(tree.h, m.ft, m.fc, m.mt, m.mc, rays, n, bgp, rgb, a, d, st):
            raise self._err()
        return rgb, a, d, st

    def render_frame(self, tree, m, cam, w, h, bg=None):
        rgb, a, d = np.zeros(w * h * 3, np.float32), np.zeros(w * h, np.float32), np.zeros(w * h, np.float32)
        st = np.zeros(5, np.int64)
        bga = _f32(bg) if bg is not None else None
        if self.lib.or_render_frame(tree.h, m.ft, m.fc, m.mt, m.mc, _f64(cam), w, h,
                                    bga.ctypes.data if bga is not None else None, rgb, a, d, st):
            raise self._err()
        return rgb, a, d, st

    def loss(self, tree, m, rays, cgt, depth, alpha, mode, lw=(1.0, 0.01, 0.01, 0.1), frozen=False, grads=True):
        rays = _f64(rays).reshape(-1, 6)
        n = rays.shape[0]
        g = Model(np.zeros_like(m.ft), np.zeros_like(m.fc), np.zeros_like(m.mt), np.zeros_like(m.mc)) if grads else None
        st = np.zeros(3, np.int64)
        loss = C.c_double()
        ptr = (lambda a: a.ctypes.data) if grads else (lambda a: None)
        rc = self.lib.or_loss(tree.h, m.ft, m.fc, m.mt, m.mc, rays, _f32(cgt).reshape(-1), _f64(depth),
                              np.ascontiguousarray(alpha, dtype=np.uint8), n, mode, _f64(lw), int(frozen),
                              ptr(g.ft) if g else None, ptr(g.fc) if g else None,
                              ptr(g.mt) if g else None, ptr(g.mc) if g else None, st, C.byref(loss))
        if rc:
            raise self._err()
        return loss.value, g, st

    def adam_step(self, params, grads, m, v, step, lr):
        self.lib.or_adam_step(params, _f32(grads), m, v, params.size, step, lr)


def _box(v):
    return None if v is None else _f64(v).ctypes.data


class OTree:
    def __init__(self, lib, h, res, dilation, lo, hi):
        self.o, self.h, self.res, self.dilation = lib, h, res, dilation
        self.lo = (0.0, 0.0, 0.0) if lo is None else tuple(lo)
        self.hi = (1.0, 1.0, 1.0) if hi is None else tuple(hi)

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.or_tree_free(self.h)
            self.h = None

    @property
    def leaf_level(self):
        return self.o.lib.or_tree_leaf_level(self.h)

    def level_codes(self, level):
        n = self.o.lib.or_tree_level_size(self.h, level)
        p = self.o.lib.or_tree_level_codes(self.h, level)
        return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint64)

    @property
    def leaf_codes(self):
        return self.level_codes(self.leaf_level)

    @property
    def corner_ids(self):
        n = self.o.lib.or_tree_level_size(self.h, self.leaf_level)
        return np.ctypeslib.as_array(self.o.lib.or_tree_corner_ids(self.h), shape=(n * 8,)).copy()

    @property
    def vertex_count(self):
        return self.o.lib.or_tree_vertex_count(self.h)

    @property
    def dropped(self):
        return self.o.lib.or_tree_dropped(self.h)

    def locate(self, p):
        c = C.c_uint64()
        return c.value if self.o.lib.or_tree_locate(self.h, _f64(p), C.byref(c)) else None


class OScene:
    def __init__(self, lib, h):
        self.o, self.h = lib, h

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.or_scene_free(self.h)
            self.h = None


class Reference:
    """The unmodified reference behind oracle/ref/ref_shim.cpp (oracle/_ref)."""

    kind = "reference"

    def __init__(self, nofma: bool = False):
        path = REF_NOFMA_SO if nofma else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_octree_build.restype = C.c_void_p
        L.ref_octree_build.argtypes = [_dp, C.c_size_t, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
        L.ref_octree_from_leaves.restype = C.c_void_p
        L.ref_octree_from_leaves.argtypes = [_u64p, C.c_size_t, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
        L.ref_octree_free.argtypes = [C.c_void_p]
        L.ref_octree_leaf_level.argtypes = [C.c_void_p]
        L.ref_octree_vertex_count.restype = C.c_uint32
        L.ref_octree_vertex_count.argtypes = [C.c_void_p]
        L.ref_octree_dropped.restype = C.c_size_t
        L.ref_octree_dropped.argtypes = [C.c_void_p]
        L.ref_octree_level_size.restype = C.c_size_t
        L.ref_octree_level_size.argtypes = [C.c_void_p, C.c_int]
        L.ref_octree_level_codes.argtypes = [C.c_void_p, C.c_int, _u64p]
        L.ref_octree_corner_ids.argtypes = [C.c_void_p, _u32p]
        L.ref_octree_locate.argtypes = [C.c_void_p, _dp, C.POINTER(C.c_uint64)]
        L.ref_traverse.restype = C.c_size_t
        L.ref_traverse.argtypes = [C.c_void_p, _dp, C.c_size_t, _u64p, C.c_size_t, _u64p, _dp, _dp, C.c_void_p]
        L.ref_ray_aabb.argtypes = [_dp, _dp, _dp, _dp]
        L.ref_camera_rays.argtypes = [_dp, C.c_uint32, C.c_uint32, _dp]
        L.ref_lookat_camera.argtypes = [_dp, _dp, C.c_uint32, C.c_uint32, C.c_double, _dp]
        L.ref_model_init.restype = C.c_void_p
        L.ref_model_init.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_sizes.restype = C.c_size_t
        L.ref_model_sizes.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(dtype=np.uintp)]
        L.ref_model_get.argtypes = [C.c_void_p, _fp, _fp, _fp, _fp]
        L.ref_model_set.argtypes = [C.c_void_p, _fp, _fp, _fp, _fp]
        L.ref_render_frame.argtypes = [C.c_void_p, _dp, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, _i64p, C.c_int, C.POINTER(C.c_double)]
        L.ref_loss.argtypes = [C.c_void_p, _dp, _fp, _dp, _u8p, C.c_size_t, C.c_int, _dp, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _i64p, C.POINTER(C.c_double)]
        L.ref_adam_step.argtypes = [_fp, _fp, _fp, _fp, C.c_size_t, C.c_uint64, C.c_float]
        L.ref_scene_make.restype = C.c_void_p
        L.ref_scene_make.argtypes = [C.c_uint64, C.c_int]
        L.ref_scene_free.argtypes = [C.c_void_p]
        L.ref_hemisphere_cameras.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, _dp]
        L.ref_scene_render_gt.argtypes = [C.c_void_p, _dp, C.c_uint32, C.c_uint32, _fp, _fp, _fp]
        L.ref_train.argtypes = [C.c_void_p, _dp, C.c_int, C.c_uint32, C.c_uint32, np.ctypeslib.ndpointer(dtype=np.int32),
                                C.c_uint32, C.c_uint32, C.c_uint64, _dp, C.c_int, C.POINTER(C.c_int), C.c_void_p]
        L.ref_thread_count.restype = C.c_int
        L.ref_train2.argtypes = [C.c_void_p, _dp, np.ctypeslib.ndpointer(dtype=np.int32), C.c_int, C.c_uint32,
                                 C.c_uint32, np.ctypeslib.ndpointer(dtype=np.int32), C.c_uint32, C.c_uint32,
                                 C.c_uint64, _dp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_longlong),
                                 C.POINTER(C.c_void_p)]

    def _err(self):
        return OracleError(self.lib.ref_last_error().decode())

    def set_threads(self, n):
        self.lib.ref_set_threads(n)

    def thread_count(self):
        return self.lib.ref_thread_count()

    def metrics(self, pred, gt, w, h, channels):
        """(psnr, ssim) of the reference (src/metrics.cpp:57-113) on interleaved float images."""
        a = np.ascontiguousarray(pred, dtype=np.float32).reshape(-1)
        b = np.ascontiguousarray(gt, dtype=np.float32).reshape(-1)
        p, q = C.c_double(), C.c_double()
        self.lib.ref_metrics.argtypes = [_fp, _fp, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
        if self.lib.ref_metrics(a, b, w, h, channels, C.byref(p), C.byref(q)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return p.value, q.value

    def tree_build(self, points, res, dilation=1, lo=None, hi=None):
        pts = _f64(points).reshape(-1, 3)
        h = self.lib.ref_octree_build(pts, pts.shape[0], res, dilation, _box(lo), _box(hi))
        if not h:
            raise self._err()
        return RTree(self, h, res, dilation, lo, hi)

    def tree_from_leaves(self, codes, res, dilation=1, lo=None, hi=None):
        c = np.ascontiguousarray(codes, dtype=np.uint64)
        h = self.lib.ref_octree_from_leaves(c, c.size, res, dilation, _box(lo), _box(hi))
        if not h:
            raise self._err()
        return RTree(self, h, res, dilation, lo, hi)

    def ray_aabb(self, ray6, lo, hi):
        t = np.zeros(2)
        ok = self.lib.ref_ray_aabb(_f64(ray6), _f64(lo), _f64(hi), t)
        return (t[0], t[1]) if ok else None

    def traverse(self, tree, rays, with_points=False):
        rays = _f64(rays).reshape(-1, 6)
        n = rays.shape[0]
        off = np.zeros(n + 1, dtype=np.uint64)
        e64, ed = np.zeros(1, np.uint64), np.zeros(1)
        total = self.lib.ref_traverse(tree.h, rays, n, off, 0, e64, ed, ed, None)
        m = max(total, 1)
        ids, tin, tout = np.zeros(m, np.uint64), np.zeros(m), np.zeros(m)
        x12 = np.zeros((m, 6)) if with_points else None
        self.lib.ref_traverse(tree.h, rays, n, off, total, ids, tin, tout,
                              x12.ctypes.data if with_points else None)
        res = (off.astype(np.int64), ids[:total], tin[:total], tout[:total])
        return res + (x12[:total],) if with_points else res

    def camera_rays(self, cam, w, h):
        out = np.zeros((w * h, 6))
        self.lib.ref_camera_rays(_f64(cam), w, h, out)
        return out

    def lookat_camera(self, eye, target, w, h, focal):
        out = np.zeros(20)
        self.lib.ref_lookat_camera(_f64(eye), _f64(target), w, h, focal, out)
        return out

    def hemisphere_cameras(self, n, radius, seed, w, h, focal):
        out = np.zeros((n, 20))
        self.lib.ref_hemisphere_cameras(n, radius, seed, w, h, focal, out)
        return out

    def scene_make(self, seed, prims):
        return RScene(self, self.lib.ref_scene_make(seed, prims))

    def scene_render_gt(self, scene, cam, w, h):
        rgb = np.zeros(w * h * 3, np.float32)
        depth = np.zeros(w * h, np.float32)
        mask = np.zeros(w * h, np.float32)
        self.lib.ref_scene_render_gt(scene.h, _f64(cam), w, h, rgb, depth, mask)
        return rgb, depth, mask

    def init_model(self, tree, seed):
        h = self.lib.ref_model_init(tree.h, seed)
        sz = np.zeros(4, dtype=np.uintp)
        self.lib.ref_model_sizes(h, sz)
        m = Model(np.zeros(sz[0], np.float32), np.zeros(sz[1], np.float32),
                  np.zeros(sz[2], np.float32), np.zeros(sz[3], np.float32))
        self.lib.ref_model_get(h, m.ft, m.fc, m.mt, m.mc)
        self.lib.ref_model_free(h)
        return m

    def train(self, scene, cams, splits, w, h, epochs, grid_res, dilation, seed):
        """train() (src/train.cpp:364-527) on views rendered by the reference's GT ray caster:
        returns (log rows [stage, epoch, mean_loss, val_psnr, seconds], skipped rays, Model)."""
        cams = _f64(cams).reshape(-1, 20)
        log = np.zeros((256, 5))
        n_log, skipped, mh = C.c_int(), C.c_longlong(), C.c_void_p()
        if self.lib.ref_train2(scene.h, cams, np.ascontiguousarray(splits, dtype=np.int32), cams.shape[0], w, h,
                               np.ascontiguousarray(epochs, dtype=np.int32), grid_res, dilation, seed, log, 256,
                               C.byref(n_log), C.byref(skipped), C.byref(mh)):
            raise self._err()
        sz = np.zeros(4, dtype=np.uintp)
        self.lib.ref_model_sizes(mh, sz)
        m = Model(np.zeros(sz[0], np.float32), np.zeros(sz[1], np.float32),
                  np.zeros(sz[2], np.float32), np.zeros(sz[3], np.float32))
        self.lib.ref_model_get(mh, m.ft, m.fc, m.mt, m.mc)
        self.lib.ref_model_free(mh)
        return log[:n_log.value], skipped.value, m

    def _with_model(self, tree, m):
        h = self.lib.ref_model_init(tree.h, 0)
        self.lib.ref_model_set(h, m.ft, m.fc, m.mt, m.mc)
        return h

    def render_frame(self, tree, m, cam, w, h, bg=None, parallel=True):
        rgb, a, d = np.zeros(w * h * 3, np.float32), np.zeros(w * h, np.float32), np.zeros(w * h, np.float32)
        st = np.zeros(5, np.int64)
        secs = C.c_double()
        bga = _f32(bg) if bg is not None else None
        hm = self._with_model(tree, m)
        try:
            rc = self.lib.ref_render_frame(hm, _f64(cam), w, h, bga.ctypes.data if bga is not None else None,
                                           rgb.ctypes.data, a.ctypes.data, d.ctypes.data, st, int(parallel),
                                           C.byref(secs))
        finally:
            self.lib.ref_model_free(hm)
        if rc:
            raise self._err()
        self.last_seconds = secs.value
        return rgb, a, d, st

    def time_render(self, model_handle, cam, w, h, parallel=True):
        secs = C.c_double()
        st = np.zeros(5, np.int64)
        if self.lib.ref_render_frame(model_handle, _f64(cam), w, h, None, None, None, None, st,
                                     int(parallel), C.byref(secs)):
            raise self._err()
        return secs.value, st

    def loss(self, tree, m, rays, cgt, depth, alpha, mode, lw=(1.0, 0.01, 0.01, 0.1), frozen=False, grads=True):
        rays = _f64(rays).reshape(-1, 6)
        n = rays.shape[0]
        g = Model(np.zeros_like(m.ft), np.zeros_like(m.fc), np.zeros_like(m.mt), np.zeros_like(m.mc)) if grads else None
        st = np.zeros(3, np.int64)
        loss = C.c_double()
        hm = self._with_model(tree, m)
        try:
            rc = self.lib.ref_loss(hm, rays, _f32(cgt).reshape(-1), _f64(depth),
                                   np.ascontiguousarray(alpha, dtype=np.uint8), n, mode, _f64(lw), int(frozen),
                                   g.ft.ctypes.data if g else None, g.fc.ctypes.data if g else None,
                                   g.mt.ctypes.data if g else None, g.mc.ctypes.data if g else None,
                                   st, C.byref(loss))
        finally:
            self.lib.ref_model_free(hm)
        if rc:
            raise self._err()
        return loss.value, g, st

    def adam_step(self, params, grads, m, v, step, lr):
        self.lib.ref_adam_step(params, _f32(grads), m, v, params.size, step, lr)


class RTree(OTree):
    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.ref_octree_free(self.h)
            self.h = None

    @property
    def leaf_level(self):
        return self.o.lib.ref_octree_leaf_level(self.h)

    def level_codes(self, level):
        n = self.o.lib.ref_octree_level_size(self.h, level)
        out = np.zeros(n, np.uint64)
        if n:
            self.o.lib.ref_octree_level_codes(self.h, level, out)
        return out

    @property
    def corner_ids(self):
        n = self.o.lib.ref_octree_level_size(self.h, self.leaf_level)
        out = np.zeros(n * 8, np.uint32)
        self.o.lib.ref_octree_corner_ids(self.h, out)
        return out

    @property
    def vertex_count(self):
        return self.o.lib.ref_octree_vertex_count(self.h)

    @property
    def dropped(self):
        return self.o.lib.ref_octree_dropped(self.h)

    def locate(self, p):
        c = C.c_uint64()
        return c.value if self.o.lib.ref_octree_locate(self.h, _f64(p), C.byref(c)) else None


class RScene(OScene):
    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.ref_scene_free(self.h)
            self.h = None


def reference_available(nofma: bool = False) -> bool:
    return os.path.exists(REF_NOFMA_SO if nofma else REF_SO)


# ---- synthetic workloads -------------------

def random_occupancy_points(res, density, seed, o=None):
    """tests/test_octree.cpp:38-48: cell centers kept with probability density."""
    o = o or Oracle()
    # uniform() stream of Rng(seed) in (z, y, x) order
    n = res ** 3
    u = _rng_uniform_stream(o, seed, n)
    idx = np.nonzero(u < density)[0]
    z, rem = np.divmod(idx, res * res)
    y, x = np.divmod(rem, res)
    h = 1.0 / res
    return np.stack([(x + 0.5) * h, (y + 0.5) * h, (z + 0.5) * h], axis=1)


def _rng_uniform_stream(o, seed, n):
    """Rng(seed).uniform() x n via the C restatement (MT19937-64 + 53-bit mapping)."""
    lib = o.lib
    if not hasattr(lib, "_stream_bound"):
        lib.or_rng_uniform_stream.argtypes = [C.c_uint64, C.c_size_t, _dp]
        lib._stream_bound = True
    out = np.zeros(n)
    lib.or_rng_uniform_stream(seed, n, out)
    return out


def random_rays(seed, n, o=None):
    """tests/test_octree.cpp:50-64 random_ray() x n from one Rng(seed)."""
    o = o or Oracle()
    lib = o.lib
    if not hasattr(lib, "_rays_bound"):
        lib.or_random_rays.argtypes = [C.c_uint64, C.c_size_t, _dp]
        lib._rays_bound = True
    out = np.zeros((n, 6))
    lib.or_random_rays(seed, n, out)
    return out


def ssim(pred, gt, w, h, channels):
    """Restatement of ssim (src/metrics.cpp:70-113) in fp64 numpy: per channel,
    separable 11-tap Gaussian (sigma 1.5, gaussian_kernel :21-32) over the
    valid region (blur_valid :35-54, horizontal then vertical), the SSIM map
    with C1 = 0.01^2, C2 = 0.03^2 and its mean; channels averaged."""
    if w < 11 or h < 11:
        raise ValueError("image smaller than the SSIM window")
    k = np.exp(-((np.arange(11) - 5.0) ** 2) / (2.0 * 1.5 * 1.5))
    k = k / k.sum()
    a = np.asarray(pred, np.float32).reshape(h, w, channels).astype(np.float64)
    b = np.asarray(gt, np.float32).reshape(h, w, channels).astype(np.float64)

    def blur(p):
        t = sum(k[i] * p[:, i:w - 10 + i] for i in range(11))
        return sum(k[i] * t[i:h - 10 + i, :] for i in range(11))

    c1, c2 = 0.01 ** 2, 0.03 ** 2
    total = 0.0
    for ch in range(channels):
        x, y = a[:, :, ch], b[:, :, ch]
        mx, my, mxx, myy, mxy = blur(x), blur(y), blur(x * x), blur(y * y), blur(x * y)
        vx, vy, cov = mxx - mx * mx, myy - my * my, mxy - mx * my
        m = ((2 * mx * my + c1) * (2 * cov + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))
        total += m.mean()
    return total / channels
