"""B200-native SVLF per-ray render + train path (arXiv 2205.07058).

Python mirror of the reference's C++ interface for this path, over the C ABI
in include/svlf_b200.h (libsvlf_b200.so, built in-tree for sm_100a):

    SparseOctree.build(points, GridConfig) / SparseOctree.from_leaves(...)
        -> reference SparseOctree::build / from_leaves (include/svlf/octree.hpp:47,82)
    octree.traverse(rays)                  -> SparseOctree::traverse (octree.hpp:75-78), batched
    Model(octree).init(seed)               -> init_model (include/svlf/model.hpp:80)
    render_frame(model, camera, ...)       -> render_frame (include/svlf/render.hpp:104-105)
    train_step(model, batch, ...)          -> the per-frame body of train() (src/train.cpp:443-479)
    loss_grads(model, batch, ...)          -> surface_loss / volumetric_loss summed (train.hpp:60-71)

Errors re-raise the reference's exception type and message (ValueError for
std::invalid_argument, RuntimeError for std::runtime_error, IndexError for
std::out_of_range). There is no CPU fallback: without the built library or a
CUDA device every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "GridConfig", "Camera", "LossWeights", "RenderStats", "LossStats", "Context", "SparseOctree",
    "Model", "render_frame", "render_rays", "train_step", "loss_grads", "library_path", "load_library",
    "DEC_T_SIZE", "DEC_C_SIZE", "SvlfCudaError",
]

HERE = os.path.dirname(os.path.abspath(__file__))
DEC_T_SIZE = 17538
DEC_C_SIZE = 38403
FEAT_T_DIM = 64
FEAT_C_DIM = 32


class SvlfCudaError(RuntimeError):
    """Device failure (no reference analogue)."""


class SvlfCapacityError(RuntimeError):
    pass


# ---- ABI structs -----------------------------------------------------------
class _Grid(C.Structure):
    _fields_ = [("resolution", C.c_uint32), ("dilation", C.c_uint32), ("lo", C.c_double * 3),
                ("hi", C.c_double * 3)]


class _Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("camera_to_world", C.c_double * 16), ("width", C.c_uint32), ("height", C.c_uint32)]


class _RenderStats(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in
                ("rays", "rays_with_hits", "traversal_hits", "thickness_queries", "color_queries")]


class _LossWeights(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("eta", "tau", "empty", "alpha")]


class _LossStats(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in ("rays", "skipped_rays", "eta_skipped")]


class _SceneDesc(C.Structure):
    _fields_ = [("spheres", C.c_void_p), ("n_spheres", C.c_size_t), ("boxes", C.c_void_p), ("n_boxes", C.c_size_t),
                ("light_dir", C.c_double * 3), ("light_rgb", C.c_double * 3), ("ambient", C.c_double * 3),
                ("background", C.c_double * 3)]


class _OctreeInfo(C.Structure):
    _fields_ = [("leaf_level", C.c_int), ("vertex_count", C.c_uint32), ("leaf_count", C.c_size_t),
                ("dropped_points", C.c_size_t), ("cell_size", C.c_double), ("level_size", C.c_size_t * 22)]


class _Timings(C.Structure):
    _fields_ = [(n, C.c_float) for n in
                ("traverse_ms", "emit_ms", "decode_ms", "composite_ms", "backward_ms", "adam_ms", "total_ms")] + \
               [("hits", C.c_longlong), ("overflow_rays", C.c_longlong), ("dense_rays", C.c_longlong)]


# ---- public value types (reference structs) ----------------------------------
@dataclass
class GridConfig:
    """include/svlf/octree.hpp:13-19."""
    resolution: int = 128
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    dilation: int = 1

    def _c(self):
        return _Grid(self.resolution, self.dilation, (C.c_double * 3)(*self.lo), (C.c_double * 3)(*self.hi))


@dataclass
class Camera:
    """include/svlf/camera.hpp:12-33; camera_to_world row-major 4x4."""
    fx: float
    fy: float
    cx: float
    cy: float
    camera_to_world: tuple
    width: int
    height: int

    @staticmethod
    def from_record(rec, width, height):
        """rec = (fx, fy, cx, cy, c2w[16]) as produced by synthetic/oracle helpers."""
        rec = [float(x) for x in rec]
        return Camera(rec[0], rec[1], rec[2], rec[3], tuple(rec[4:20]), int(width), int(height))

    def record(self):
        return np.array([self.fx, self.fy, self.cx, self.cy, *self.camera_to_world], dtype=np.float64)

    def _c(self):
        return _Camera(self.fx, self.fy, self.cx, self.cy, (C.c_double * 16)(*self.camera_to_world),
                       self.width, self.height)


@dataclass
class LossWeights:
    """include/svlf/train.hpp:43-48."""
    eta: float = 1.0
    tau: float = 0.01
    empty: float = 0.01
    alpha: float = 0.1

    def _c(self):
        return _LossWeights(self.eta, self.tau, self.empty, self.alpha)


@dataclass
class RenderStats:
    """include/svlf/render.hpp:94-100."""
    rays: int = 0
    rays_with_hits: int = 0
    traversal_hits: int = 0
    thickness_queries: int = 0
    color_queries: int = 0


@dataclass
class LossStats:
    """include/svlf/train.hpp:50-54."""
    rays: int = 0
    skipped_rays: int = 0
    eta_skipped: int = 0


# ---- library loading -----------------------------------------------------------
_LIB = None
# int (*)(void* user, void* host_buf, size_t count, svlf_dtype, svlf_reduce_op)
_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int)


def library_path() -> str:
    # $SVLF_LIB_PATH: an alternative build of the same library (tuning experiments)
    return os.environ.get("SVLF_LIB_PATH") or os.path.join(HERE, "libsvlf_b200.so")


def _dp(a):
    return a.ctypes.data_as(C.c_void_p)


def load_library():
    """Load libsvlf_b200.so (fails loudly when it is missing: no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = library_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run __graft_entry__.build() (make -C paper_2205_07058_b200/csrc)")
    L = C.CDLL(path)
    vp, sz, st = C.c_void_p, C.c_size_t, C.c_int
    sigs = {
        "svlf_last_error": ([], C.c_char_p),
        "svlf_abi_version": ([], C.c_int),
        "svlf_ctx_create": ([C.c_int, C.POINTER(vp)], st),
        "svlf_ctx_destroy": ([vp], st),
        "svlf_ctx_synchronize": ([vp], st),
        "svlf_ctx_set_stream": ([vp, vp], st),
        "svlf_ctx_last_timings": ([vp, C.POINTER(_Timings)], st),
        "svlf_ctx_kernel_launches": ([vp], C.c_longlong),
        "svlf_render_frame_submit": ([vp, vp, vp, vp, C.c_int, vp, vp, vp, C.POINTER(C.c_uint64)], st),
        "svlf_render_frame_wait": ([vp, C.c_uint64, vp], st),
        "svlf_render_gt_device": ([vp, vp, vp, vp, vp, vp], st),
        "svlf_backproject_device": ([vp, vp, vp, vp, sz, C.POINTER(sz)], st),
        "svlf_psnr_device": ([vp, vp, vp, sz, C.POINTER(C.c_double)], st),
        "svlf_ctx_last_node_tests": ([vp, C.POINTER(C.c_longlong)], st),
        "svlf_ctx_set_node_test_counting": ([vp, C.c_int], st),
        "svlf_ssim_device": ([vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_double)], st),
        "svlf_depth_errors_device": ([vp, vp, vp, vp, sz, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int)], st),
        "svlf_host_alloc": ([sz, vp], st),
        "svlf_host_free": ([vp], st),
        "svlf_ctx_set_train_precision": ([vp, C.c_int], st),
        "svlf_nccl_unique_id": ([vp], st),
        "svlf_ctx_attach_nccl": ([vp, vp, C.c_int, C.c_int], st),
        "svlf_ctx_detach_nccl": ([vp], st),
        "svlf_ctx_attach_collective": ([vp, _ALLREDUCE_FN, vp, C.c_int, C.c_int], st),
        "svlf_model_set_adam_hyper": ([vp, vp, vp, vp], st),
        "svlf_model_get_adam_hyper": ([vp, vp, vp, vp], st),
        "svlf_octree_build": ([vp, C.POINTER(_Grid), vp, sz, C.POINTER(vp)], st),
        "svlf_octree_build_device": ([vp, C.POINTER(_Grid), vp, sz, C.POINTER(vp)], st),
        "svlf_octree_from_leaves": ([vp, C.POINTER(_Grid), vp, sz, C.POINTER(vp)], st),
        "svlf_octree_destroy": ([vp], st),
        "svlf_octree_get_info": ([vp, C.POINTER(_OctreeInfo)], st),
        "svlf_octree_level_codes": ([vp, C.c_int, vp], st),
        "svlf_octree_corner_ids": ([vp, vp], st),
        "svlf_traverse": ([vp, vp, vp, sz, vp, sz, vp, vp, vp, vp, C.POINTER(sz)], st),
        "svlf_model_create": ([vp, vp, C.POINTER(vp)], st),
        "svlf_model_destroy": ([vp], st),
        "svlf_model_init": ([vp, C.c_uint64], st),
        "svlf_model_set_params": ([vp, vp, vp, vp, vp], st),
        "svlf_model_get_params": ([vp, vp, vp, vp, vp], st),
        "svlf_model_get_grads": ([vp, vp, vp, vp, vp], st),
        "svlf_model_get_adam": ([vp, vp, vp, vp], st),
        "svlf_model_set_adam": ([vp, vp, vp, vp], st),
        "svlf_model_param_count": ([vp], sz),
        "svlf_render_frame": ([vp, vp, C.POINTER(_Camera), vp, C.c_int, vp, vp, vp, C.POINTER(_RenderStats)], st),
        "svlf_render_frame_device": ([vp, vp, C.POINTER(_Camera), vp, C.c_int, vp, vp, vp,
                                      C.POINTER(_RenderStats)], st),
        "svlf_render_frame_device_submit": ([vp, vp, C.POINTER(_Camera), vp, C.c_int, vp, vp, vp], st),
        "svlf_render_frame_device_finish": ([vp, C.POINTER(_RenderStats)], st),
        "svlf_local_coords": ([vp, vp, vp, vp, sz, vp], st),
        "svlf_interpolate": ([vp, vp, C.c_int, vp, C.c_uint32, C.c_uint32, vp, vp, sz, vp], st),
        "svlf_interpolate_backward": ([vp, vp, C.c_int, vp, C.c_uint32, C.c_uint32, vp, vp, sz, vp, vp, vp], st),
        "svlf_parameterize_rays": ([vp, vp, vp, sz, vp], st),
        "svlf_composite": ([vp, vp, sz, vp, vp, vp, vp, vp, vp, vp], st),
        "svlf_evaluate_voxels": ([vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp], st),
        "svlf_eta_gt": ([vp, vp, vp, vp, sz, vp], st),
        "svlf_render_tiles_device": ([vp, vp, C.POINTER(_Camera), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                      vp, C.c_int, vp, vp, vp, C.POINTER(_RenderStats)], st),
        "svlf_tiles_owned": ([C.POINTER(_Camera), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32], sz),
        "svlf_render_rows_device": ([vp, vp, C.POINTER(_Camera), C.c_uint32, C.c_uint32, vp, C.c_int, vp, vp, vp,
                                     C.POINTER(_RenderStats)], st),
        "svlf_render_rays": ([vp, vp, vp, sz, vp, C.c_int, vp, vp, vp, C.POINTER(_RenderStats)], st),
        "svlf_train_step": ([vp, vp, vp, vp, vp, vp, sz, C.c_int, C.c_int, C.c_float, C.POINTER(_LossWeights),
                             C.POINTER(_LossStats), C.POINTER(C.c_double)], st),
        "svlf_train_step_device": ([vp, vp, vp, vp, vp, vp, sz, C.c_int, C.c_int, C.c_float,
                                    C.POINTER(_LossWeights), C.POINTER(_LossStats), C.POINTER(C.c_double)], st),
        "svlf_train_batch_stage": ([vp, vp, vp, vp, vp, sz, C.POINTER(C.c_int)], st),
        "svlf_train_step_staged": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_float, C.POINTER(_LossWeights),
                                    C.POINTER(_LossStats), C.POINTER(C.c_double)], st),
        "svlf_train_batch_discard": ([vp, C.c_int], st),
        "svlf_loss_grads": ([vp, vp, vp, vp, vp, vp, sz, C.c_int, C.c_int, C.POINTER(_LossWeights),
                             C.POINTER(_LossStats), C.POINTER(C.c_double)], st),
    }
    for name, (args, res) in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _LIB = L
    return L


def _check(status):
    if status == 0:
        return
    msg = _LIB.svlf_last_error().decode()
    if status == 1:
        raise ValueError(msg)
    if status == 3:
        raise IndexError(msg)
    if status == 4:
        raise SvlfCudaError(msg)
    if status == 5:
        raise SvlfCapacityError(msg)
    raise RuntimeError(msg)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---- objects ------------------------------------------------------------------
class Context:
    """One CUDA device + stream + scratch arenas (svlf_ctx)."""

    def __init__(self, device: int = 0):
        L = load_library()
        h = C.c_void_p()
        _check(L.svlf_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self._deps = weakref.WeakSet()  # models bound to this context

    @property
    def handle(self):
        return self._h

    def close(self):
        """Destroys the context; models created on it are released first."""
        if getattr(self, "_h", None):
            for dep in list(getattr(self, "_deps", ())):
                dep._release()
            _LIB.svlf_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(_LIB.svlf_ctx_synchronize(self._h))

    def set_stream(self, stream_ptr: int | None):
        _check(_LIB.svlf_ctx_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def last_timings(self) -> dict:
        t = _Timings()
        _check(_LIB.svlf_ctx_last_timings(self._h, C.byref(t)))
        return {n: getattr(t, n) for n, _ in _Timings._fields_}

    def set_node_test_counting(self, enable: bool):
        """Diagnostics: run the traversal variant that counts ray-box tests (see last_node_tests)."""
        _check(_LIB.svlf_ctx_set_node_test_counting(self._h, 1 if enable else 0))

    def last_node_tests(self) -> int:
        """Ray-box tests of the last traversal's cooperative passes (reference ray_aabb calls)."""
        v = C.c_longlong()
        _check(_LIB.svlf_ctx_last_node_tests(self._h, C.byref(v)))
        return int(v.value)

    @staticmethod
    def kernel_launches() -> int:
        return int(load_library().svlf_ctx_kernel_launches(None))

    def set_train_precision(self, precision: str):
        """Dense-layer GEMMs of the train step, all on this library's tcgen05 kernels:
        'fp32' (default) / 'tf32x3' (three TF32 products of split operands: fp32-level
        accuracy, deterministic) or 'tf32' (weight-gradient reductions with plain TF32
        operands: 16-bit tolerance)."""
        _check(_LIB.svlf_ctx_set_train_precision(self._h, {**_PREC, "tf32": 3, "tf32x3": 4}[precision]))

    def attach_nccl(self, unique_id: bytes, rank: int, world: int):
        """Data-parallel training: all-reduce loss, statistics and gradients over NCCL."""
        _load_framework_nccl()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(_LIB.svlf_ctx_attach_nccl(self._h, buf, rank, world))

    def detach_nccl(self):
        _check(_LIB.svlf_ctx_detach_nccl(self._h))

    def attach_host_collective(self, allreduce, rank: int, world: int):
        """Data-parallel training over a host-side all-reduce instead of NCCL:
        `allreduce(buf, op)` reduces the numpy array `buf` in place across the
        ranks (op 'sum' or 'max'); e.g. torch.distributed over gloo
        (parallel.init_data_parallel_host)."""
        dtypes = {0: np.float32, 1: np.float64, 2: np.uint8}

        def tramp(_user, ptr, count, dtype, op):
            try:
                dt = np.dtype(dtypes[dtype])
                buf = np.frombuffer((C.c_char * (count * dt.itemsize)).from_address(ptr), dtype=dt, count=count)
                allreduce(buf, "sum" if op == 0 else "max")
                return 0
            except BaseException:  # noqa: BLE001 - reported to the library as a failed exchange
                import traceback
                traceback.print_exc()
                return 1

        cb = _ALLREDUCE_FN(tramp)
        _check(_LIB.svlf_ctx_attach_collective(self._h, cb, None, rank, world))
        self._collective_cb = cb  # kept alive with the context


class _PinnedBlock:
    """Page-locked host allocation (svlf_host_alloc); freed with the last view."""

    def __init__(self, nbytes: int):
        load_library()
        h = C.c_void_p()
        _check(_LIB.svlf_host_alloc(nbytes, C.byref(h)))
        self.ptr = h.value
        self.nbytes = nbytes

    def __del__(self):
        if getattr(self, "ptr", None) and _LIB is not None:
            _LIB.svlf_host_free(C.c_void_p(self.ptr))
            self.ptr = None


def pinned_empty(n: int, dtype=np.float32) -> np.ndarray:
    """1-D numpy array of n elements in page-locked host memory."""
    dt = np.dtype(dtype)
    block = _PinnedBlock(max(1, n * dt.itemsize))
    buf = (C.c_char * block.nbytes).from_address(block.ptr)
    arr = np.frombuffer(buf, dtype=dt, count=n)
    weakref.finalize(arr, lambda b: None, block)  # keep the block alive with the array
    return arr


def pinned_frame(width: int, height: int):
    """(rgb, alpha, depth) output buffers in page-locked memory for render_frame(out=...):
    the frame's device-to-host copies then land in them directly."""
    n = width * height
    return pinned_empty(3 * n), pinned_empty(n), pinned_empty(n)


def _load_framework_nccl():
    # The library resolves NCCL with dlopen("libnccl.so.2"): make sure PyTorch's
    # bundled NCCL is the one in the process (a different build loaded first
    # would break a later `import torch`).
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (create on one rank, share with the others)."""
    _load_framework_nccl()
    load_library()
    buf = C.create_string_buffer(128)
    _check(_LIB.svlf_nccl_unique_id(buf))
    return buf.raw


_DEFAULT_CTX = None


def default_context() -> Context:
    global _DEFAULT_CTX
    if _DEFAULT_CTX is None:
        _DEFAULT_CTX = Context(0)
    return _DEFAULT_CTX


class SparseOctree:
    """Host-built octree with a device mirror (reference SparseOctree)."""

    def __init__(self, handle, ctx: Context, grid: GridConfig):
        self._h = handle
        self.ctx = ctx
        self.config = grid
        info = _OctreeInfo()
        _check(_LIB.svlf_octree_get_info(self._h, C.byref(info)))
        self.leaf_level = info.leaf_level
        self.vertex_count = info.vertex_count
        self.leaf_count = info.leaf_count
        self.dropped_points = info.dropped_points
        self.cell_size = info.cell_size
        self._level_sizes = [info.level_size[i] for i in range(self.leaf_level + 1)]

    @staticmethod
    def build_device(d_points: int, n: int, grid: GridConfig, ctx: Context) -> "SparseOctree":
        """GPU build from n x 3 float64 points already in device memory (pointer as int)."""
        load_library()
        h = C.c_void_p()
        g = grid._c()
        _check(_LIB.svlf_octree_build_device(ctx.handle, C.byref(g), C.c_void_p(d_points), n, C.byref(h)))
        return SparseOctree(h, ctx, grid)

    @staticmethod
    def build(points, grid: GridConfig, ctx: Context | None = None) -> "SparseOctree":
        """With a context: GPU build (byte-identical); without: host build (no device needed,
        uploaded on first use by a context)."""
        load_library()
        pts = _f64(points).reshape(-1, 3)
        h = C.c_void_p()
        g = grid._c()
        _check(_LIB.svlf_octree_build(ctx.handle if ctx else None, C.byref(g), _dp(pts), pts.shape[0],
                                      C.byref(h)))
        return SparseOctree(h, ctx, grid)

    @staticmethod
    def from_leaves(codes, grid: GridConfig, ctx: Context | None = None) -> "SparseOctree":
        load_library()
        c = np.ascontiguousarray(codes, dtype=np.uint64)
        h = C.c_void_p()
        g = grid._c()
        _check(_LIB.svlf_octree_from_leaves(ctx.handle if ctx else None, C.byref(g), _dp(c), c.size,
                                            C.byref(h)))
        return SparseOctree(h, ctx, grid)

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.svlf_octree_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def level_codes(self, level: int) -> np.ndarray:
        out = np.zeros(self._level_sizes[level], np.uint64)
        _check(_LIB.svlf_octree_level_codes(self._h, level, _dp(out)))
        return out

    @property
    def leaf_codes(self) -> np.ndarray:
        return self.level_codes(self.leaf_level)

    def corner_ids(self) -> np.ndarray:
        out = np.zeros(self.leaf_count * 8, np.uint32)
        _check(_LIB.svlf_octree_corner_ids(self._h, _dp(out)))
        return out

    def corner_vertices(self, voxel_id: int) -> np.ndarray:
        leaves = self.leaf_codes
        i = int(np.searchsorted(leaves, np.uint64(voxel_id)))
        if i >= leaves.size or leaves[i] != np.uint64(voxel_id):
            raise IndexError("unknown voxel id")
        return self.corner_ids()[8 * i: 8 * i + 8]

    def traverse(self, rays, with_points: bool = False):
        """Batched traversal on the GPU: rays n x 6 -> (offsets[n+1], voxel_ids,
        t_in, t_out[, x12 (n_hits x 6)]), each ray's hits sorted by (t_in, id)."""
        r = _f64(rays).reshape(-1, 6)
        n = r.shape[0]
        off = np.zeros(n + 1, np.uint64)
        total = C.c_size_t(0)
        cap = max(8 * n, 1024)
        while True:
            ids = np.zeros(cap, np.uint64)
            tin = np.zeros(cap)
            tout = np.zeros(cap)
            x12 = np.zeros((cap, 6)) if with_points else None
            ctx = self.ctx or default_context()
            st = _LIB.svlf_traverse(ctx.handle, self._h, _dp(r), n, _dp(off), cap, _dp(ids), _dp(tin),
                                    _dp(tout), _dp(x12) if with_points else None, C.byref(total))
            if st == 5:
                cap = int(total.value)
                continue
            _check(st)
            break
        t = int(total.value)
        out = (off.astype(np.int64), ids[:t], tin[:t], tout[:t])
        return out + (x12[:t],) if with_points else out


class Model:
    """SvlfModel + gradients + ModelAdam, resident on the device."""

    def __init__(self, octree: SparseOctree, seed: int | None = None, ctx: Context | None = None):
        self.octree = octree
        self.ctx = ctx or octree.ctx or default_context()
        h = C.c_void_p()
        _check(_LIB.svlf_model_create(self.ctx.handle, octree.handle, C.byref(h)))
        self._h = h
        self.ctx._deps.add(self)
        self.V = octree.vertex_count
        if seed is not None:
            self.init(seed)

    def _release(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.svlf_model_destroy(self._h)
            self._h = None

    def __del__(self):
        self._release()

    @property
    def handle(self):
        return self._h

    def init(self, seed: int):
        _check(_LIB.svlf_model_init(self._h, seed))
        return self

    def _bufs(self):
        return (np.zeros(self.V * FEAT_T_DIM, np.float32), np.zeros(self.V * FEAT_C_DIM, np.float32),
                np.zeros(DEC_T_SIZE, np.float32), np.zeros(DEC_C_SIZE, np.float32))

    def set_params(self, ft=None, fc=None, mt=None, mc=None):
        arrs = [None if a is None else _f32(a).reshape(-1) for a in (ft, fc, mt, mc)]
        sizes = (self.V * FEAT_T_DIM, self.V * FEAT_C_DIM, DEC_T_SIZE, DEC_C_SIZE)
        for a, s in zip(arrs, sizes):
            if a is not None and a.size != s:
                raise ValueError("parameter size mismatch")
        _check(_LIB.svlf_model_set_params(self._h, *[None if a is None else _dp(a) for a in arrs]))

    def get_params(self):
        b = self._bufs()
        _check(_LIB.svlf_model_get_params(self._h, *[_dp(a) for a in b]))
        return b

    def get_grads(self):
        b = self._bufs()
        _check(_LIB.svlf_model_get_grads(self._h, *[_dp(a) for a in b]))
        return b

    def param_count(self) -> int:
        return int(_LIB.svlf_model_param_count(self._h))

    def get_adam(self):
        n = self.param_count()
        m, v = np.zeros(n, np.float32), np.zeros(n, np.float32)
        steps = np.zeros(14, np.uint64)
        _check(_LIB.svlf_model_get_adam(self._h, _dp(m), _dp(v), _dp(steps)))
        return m, v, steps

    def set_adam(self, m, v, steps):
        m, v = _f32(m), _f32(v)
        steps = np.ascontiguousarray(steps, dtype=np.uint64)
        _check(_LIB.svlf_model_set_adam(self._h, _dp(m), _dp(v), _dp(steps)))

    def get_adam_hyper(self):
        """(beta1, beta2, eps) of the 14 Adam tensors (AdamState fields)."""
        b1, b2, e = (np.zeros(14, np.float32) for _ in range(3))
        _check(_LIB.svlf_model_get_adam_hyper(self._h, _dp(b1), _dp(b2), _dp(e)))
        return b1, b2, e

    def set_adam_hyper(self, beta1, beta2, eps):
        arrs = [np.ascontiguousarray(np.broadcast_to(np.asarray(a, np.float32), (14,))) for a in (beta1, beta2, eps)]
        _check(_LIB.svlf_model_set_adam_hyper(self._h, *[_dp(a) for a in arrs]))


_PREC = {"fp32": 0, "bf16": 1, "fp16": 2}


def _bg(background):
    if background is None:
        return None, None
    b = _f32(background).reshape(3)
    return b, _dp(b)


def render_frame(model: Model, camera: Camera, stats: RenderStats | None = None, background=None,
                 precision: str = "fp32", out=None):
    """render_frame (include/svlf/render.hpp:104): returns (rgb HxWx3, alpha HxW, depth HxW).

    `out` = (rgb, alpha, depth) float32 C-contiguous arrays with W*H*3, W*H, W*H
    elements to render into (the reference's caller-owned FrameBuffers, reused
    across frames); fresh arrays are allocated otherwise."""
    n = camera.width * camera.height
    if out is None:
        rgb = np.empty(n * 3, np.float32)
        alpha = np.empty(n, np.float32)
        depth = np.empty(n, np.float32)
    else:
        rgb, alpha, depth = out
        for arr, k in ((rgb, 3 * n), (alpha, n), (depth, n)):
            if not (isinstance(arr, np.ndarray) and arr.dtype == np.float32 and arr.size == k
                    and arr.flags.c_contiguous and arr.flags.writeable):
                raise ValueError("out arrays must be writeable C-contiguous float32 of sizes W*H*3, W*H, W*H")
    st = _RenderStats()
    keep, bgp = _bg(background)
    cam = camera._c()
    _check(_LIB.svlf_render_frame(model.ctx.handle, model.handle, C.byref(cam), bgp, _PREC[precision],
                                  _dp(rgb), _dp(alpha), _dp(depth), C.byref(st)))
    _add_stats(stats, st)
    return (rgb.reshape(camera.height, camera.width, 3), alpha.reshape(camera.height, camera.width),
            depth.reshape(camera.height, camera.width))


# ---- ground truth / occupancy / metrics on the GPU (device pointers as ints) ----
def _scene_desc(scene):
    sp = np.array([[*c, r, *a] for c, r, a in scene.spheres], np.float64).reshape(-1, 7)
    bx = np.array([[*lo, *hi, *a] for lo, hi, a in scene.boxes], np.float64).reshape(-1, 9)
    d = _SceneDesc(sp.ctypes.data if sp.size else None, sp.shape[0], bx.ctypes.data if bx.size else None,
                   bx.shape[0], (C.c_double * 3)(*scene.light_dir), (C.c_double * 3)(*scene.light_rgb),
                   (C.c_double * 3)(*scene.ambient), (C.c_double * 3)(*scene.background))
    return d, (sp, bx)


def render_gt_device(ctx: Context, scene, camera: Camera, d_rgb: int, d_depth: int, d_mask: int):
    """Analytic-scene ground truth (raycast + shade) for every pixel into device buffers."""
    load_library()
    desc, keep = _scene_desc(scene)
    cam = camera._c()
    _check(_LIB.svlf_render_gt_device(ctx.handle, C.byref(desc), C.byref(cam), C.c_void_p(d_rgb),
                                      C.c_void_p(d_depth), C.c_void_p(d_mask)))


def backproject_device(ctx: Context, camera: Camera, d_depth: int, d_points: int, capacity: int) -> int:
    """Foreground depth -> world points (n x 3 float64) appended at d_points; returns the count."""
    n = C.c_size_t()
    cam = camera._c()
    _check(_LIB.svlf_backproject_device(ctx.handle, C.byref(cam), C.c_void_p(d_depth), C.c_void_p(d_points),
                                        capacity, C.byref(n)))
    return n.value


def psnr_device(ctx: Context, d_pred: int, d_gt: int, n_values: int) -> float:
    out = C.c_double()
    _check(_LIB.svlf_psnr_device(ctx.handle, C.c_void_p(d_pred), C.c_void_p(d_gt), n_values, C.byref(out)))
    return out.value


def ssim_device(ctx: Context, d_pred: int, d_gt: int, width: int, height: int, channels: int = 3) -> float:
    """ssim (src/metrics.cpp:70-113) of two interleaved float images on the device."""
    out = C.c_double()
    _check(_LIB.svlf_ssim_device(ctx.handle, C.c_void_p(d_pred), C.c_void_p(d_gt), width, height, channels,
                                 C.byref(out)))
    return out.value


def depth_errors_device(ctx: Context, d_pred: int, d_gt: int, d_mask: int, n_px: int):
    """(rmse, mae, empty_mask) over pixels with gt mask >= 0.5."""
    r, m, e = C.c_double(), C.c_double(), C.c_int()
    _check(_LIB.svlf_depth_errors_device(ctx.handle, C.c_void_p(d_pred), C.c_void_p(d_gt), C.c_void_p(d_mask),
                                         n_px, C.byref(r), C.byref(m), C.byref(e)))
    return r.value, m.value, bool(e.value)


class FrameTicket:
    """A submitted frame (render_frame_submit); wait() returns its buffers."""

    def __init__(self, model, camera, ticket, out, keep):
        self.model, self.camera, self.ticket, self.out, self._keep = model, camera, ticket, out, keep
        self.done = False

    def wait(self, stats: RenderStats | None = None):
        if not self.done:
            st = _RenderStats()
            _check(_LIB.svlf_render_frame_wait(self.model.ctx.handle, C.c_uint64(self.ticket), C.byref(st)))
            _add_stats(stats, st)
            self.done = True
        W, H = self.camera.width, self.camera.height
        rgb, alpha, depth = self.out
        return rgb.reshape(H, W, 3), alpha.reshape(H, W), depth.reshape(H, W)


def render_frame_submit(model: Model, camera: Camera, out, background=None, precision: str = "fp32"):
    """Pipelined render_frame: enqueue the frame (and its copies into `out`,
    ideally from pinned_frame()) and return a FrameTicket; up to two frames in
    flight per context. Call ticket.wait() before reading `out`."""
    n = camera.width * camera.height
    rgb, alpha, depth = out
    for arr, k in ((rgb, 3 * n), (alpha, n), (depth, n)):
        if not (isinstance(arr, np.ndarray) and arr.dtype == np.float32 and arr.size == k
                and arr.flags.c_contiguous and arr.flags.writeable):
            raise ValueError("out arrays must be writeable C-contiguous float32 of sizes W*H*3, W*H, W*H")
    keep, bgp = _bg(background)
    cam = camera._c()
    t = C.c_uint64()
    _check(_LIB.svlf_render_frame_submit(model.ctx.handle, model.handle, C.byref(cam), bgp, _PREC[precision],
                                         _dp(rgb), _dp(alpha), _dp(depth), C.byref(t)))
    return FrameTicket(model, camera, t.value, out, keep)


def render_frame_device(model: Model, camera: Camera, d_rgb: int, d_alpha: int, d_depth: int,
                        stats: RenderStats | None = None, background=None, precision: str = "fp32",
                        row0: int = 0, rows: int | None = None):
    """Device-buffer variant (pointers as ints); rows sub-range for tile sharding."""
    st = _RenderStats()
    keep, bgp = _bg(background)
    cam = camera._c()
    rows = camera.height - row0 if rows is None else rows
    _check(_LIB.svlf_render_rows_device(model.ctx.handle, model.handle, C.byref(cam), row0, rows, bgp,
                                        _PREC[precision], C.c_void_p(d_rgb), C.c_void_p(d_alpha),
                                        C.c_void_p(d_depth), C.byref(st)))
    _add_stats(stats, st)


def render_frame_device_submit(model: Model, camera: Camera, d_rgb: int, d_alpha: int, d_depth: int,
                               background=None, precision: str = "fp32"):
    """render_frame_device, first phase: enqueue the frame on the context's stream
    and return (16-bit modes: no host round trip). render_frame_device_finish
    completes it; the context accepts no other work until then."""
    _, bgp = _bg(background)  # the values are copied at the submit
    cam = camera._c()
    _check(_LIB.svlf_render_frame_device_submit(model.ctx.handle, model.handle, C.byref(cam), bgp,
                                                _PREC[precision], C.c_void_p(d_rgb), C.c_void_p(d_alpha),
                                                C.c_void_p(d_depth)))


def render_frame_device_finish(ctx: "Context", stats: RenderStats | None = None):
    """Second phase: wait for the submitted frame, check its counters and error
    flag, add its statistics (re-renders synchronously if the hit buffers overflowed)."""
    st = _RenderStats()
    _check(_LIB.svlf_render_frame_device_finish(ctx.handle, C.byref(st)))
    _add_stats(stats, st)


# ---- per-point / per-ray operations of the reference API (batched on the GPU) ----
def _ctx_of(ctx):
    return (ctx or default_context()).handle


def local_coords(octree: SparseOctree, voxel_ids, points, ctx: Context | None = None) -> np.ndarray:
    """local_coords (features.hpp:69) per point: n x 3."""
    ids = np.ascontiguousarray(voxel_ids, dtype=np.uint64).reshape(-1)
    p = _f64(points).reshape(-1, 3)
    u = np.zeros((ids.size, 3))
    _check(_LIB.svlf_local_coords(_ctx_of(ctx or octree.ctx), octree.handle, _dp(ids), _dp(p), ids.size, _dp(u)))
    return u


def _vol(volume):
    v = np.ascontiguousarray(volume)
    if v.dtype not in (np.float32, np.float64) or v.ndim != 2:
        raise ValueError("volume must be a rows x dim float32 / float64 array")
    return v, (0 if v.dtype == np.float32 else 1)


def interpolate(volume, octree: SparseOctree, voxel_ids, points, ctx: Context | None = None) -> np.ndarray:
    """interpolate (features.hpp:72) per point: n x dim in the volume's dtype."""
    v, dt = _vol(volume)
    ids = np.ascontiguousarray(voxel_ids, dtype=np.uint64).reshape(-1)
    p = _f64(points).reshape(-1, 3)
    out = np.zeros((ids.size, v.shape[1]), v.dtype)
    _check(_LIB.svlf_interpolate(_ctx_of(ctx or octree.ctx), octree.handle, dt, _dp(v), v.shape[0], v.shape[1],
                                 _dp(ids), _dp(p), ids.size, _dp(out)))
    return out


def interpolate_backward(volume, octree: SparseOctree, voxel_ids, points, upstream, grad_buf, with_jacobian=False,
                         ctx: Context | None = None):
    """interpolate_backward (features.hpp:76): grad_buf (rows x dim) += w * upstream in place;
    returns the positional Jacobians (n x dim x 3) when asked."""
    v, dt = _vol(volume)
    ids = np.ascontiguousarray(voxel_ids, dtype=np.uint64).reshape(-1)
    p = _f64(points).reshape(-1, 3)
    up = np.ascontiguousarray(upstream, dtype=v.dtype).reshape(ids.size, v.shape[1])
    if not (isinstance(grad_buf, np.ndarray) and grad_buf.dtype == v.dtype and grad_buf.shape == v.shape
            and grad_buf.flags.c_contiguous):
        raise ValueError("grad_buf must be a C-contiguous array shaped and typed like the volume")
    jac = np.zeros((ids.size, v.shape[1], 3)) if with_jacobian else None
    _check(_LIB.svlf_interpolate_backward(_ctx_of(ctx or octree.ctx), octree.handle, dt, _dp(v), v.shape[0],
                                          v.shape[1], _dp(ids), _dp(p), ids.size, _dp(up), _dp(grad_buf),
                                          _dp(jac) if jac is not None else None))
    return jac


def parameterize_rays(rays, boxes, ctx: Context | None = None) -> np.ndarray:
    """parameterize_ray (render.hpp:28) per (ray, box (lo xyz, hi xyz)): n x 6 (p1, p2)."""
    load_library()
    r = _f64(rays).reshape(-1, 6)
    b = _f64(boxes).reshape(-1, 6)
    out = np.zeros((r.shape[0], 6))
    _check(_LIB.svlf_parameterize_rays(_ctx_of(ctx), _dp(r), _dp(b), r.shape[0], _dp(out)))
    return out


def composite(taus, colors, t_s=None, offsets=None, ctx: Context | None = None):
    """composite (render.hpp:60) of one sample list, or of several (offsets = n_lists + 1 row
    pointer): (colour n_lists x 3, alpha, weights per sample, expected depth or None)."""
    load_library()
    t = _f64(taus).reshape(-1)
    c = _f64(colors).reshape(-1, 3)
    if c.shape[0] != t.size:
        raise ValueError("composite size mismatch")
    off = np.array([0, t.size], np.uint64) if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint64)
    nl = off.size - 1
    col, a, w = np.zeros((nl, 3)), np.zeros(nl), np.zeros(t.size)
    ts = None if t_s is None else _f64(t_s).reshape(-1)
    d = np.zeros(nl) if ts is not None else None
    _check(_LIB.svlf_composite(_ctx_of(ctx), _dp(off), nl, _dp(t), _dp(c), _dp(ts) if ts is not None else None,
                               _dp(col), _dp(a), _dp(d) if d is not None else None, _dp(w)))
    return col, a, w, d


def evaluate_voxels(model: Model, rays, voxel_ids, t_in, t_out) -> dict:
    """evaluate_voxel (render.hpp:49) per (ray, hit) with the fp32 decoders: tau, eta, x_s, t_s, color."""
    r = _f64(rays).reshape(-1, 6)
    ids = np.ascontiguousarray(voxel_ids, dtype=np.uint64).reshape(-1)
    ti, to = _f64(t_in).reshape(-1), _f64(t_out).reshape(-1)
    n = ids.size
    out = {"tau": np.zeros(n), "eta": np.zeros(n), "x_s": np.zeros((n, 3)), "t_s": np.zeros(n),
           "color": np.zeros((n, 3))}
    _check(_LIB.svlf_evaluate_voxels(model.ctx.handle, model.handle, _dp(r), _dp(ids), _dp(ti), _dp(to), n,
                                     *[_dp(out[k]) for k in ("tau", "eta", "x_s", "t_s", "color")]))
    return out


def eta_gt(t_in, t_out, depth, ctx: Context | None = None) -> np.ndarray:
    """eta_gt (train.hpp:41) per hit."""
    load_library()
    ti, to, d = (_f64(x).reshape(-1) for x in (t_in, t_out, depth))
    out = np.zeros(ti.size)
    _check(_LIB.svlf_eta_gt(_ctx_of(ctx), _dp(ti), _dp(to), _dp(d), ti.size, _dp(out)))
    return out


def render_ray(model: Model, ray) -> dict:
    """render_ray (render.hpp:75): GPU traversal, every hit through evaluate_voxel, composite;
    colour, alpha, expected depth and the samples."""
    r = _f64(ray).reshape(1, 6)
    off, ids, tin, tout = model.octree.traverse(r)
    ev = evaluate_voxels(model, np.repeat(r, ids.size, axis=0), ids, tin, tout)
    col, a, w, d = composite(ev["tau"], ev["color"], t_s=ev["t_s"], ctx=model.ctx)
    return {"color": col[0], "alpha": float(a[0]), "expected_depth": float(d[0]),
            "samples": {"voxel_ids": ids, "t_in": tin, "t_out": tout, **ev}}


def tiles_owned(camera: Camera, tile_w: int, tile_h: int, rank: int, world: int) -> int:
    """Tiles rank renders in a tile-interleaved split of the frame (0 if the tile size does not
    divide the image)."""
    load_library()
    cam = camera._c()
    return int(_LIB.svlf_tiles_owned(C.byref(cam), tile_w, tile_h, rank, world))


def render_tiles_device(model: Model, camera: Camera, tile_w: int, tile_h: int, rank: int, world: int,
                        d_rgb: int, d_alpha: int, d_depth: int, stats: RenderStats | None = None,
                        background=None, precision: str = "fp32"):
    """Rank's share of a tile-interleaved multi-GPU frame (tiles rank, rank + world, ...) into
    device buffers of tiles_owned(...) * tile_w * tile_h pixels, tile by tile."""
    st = _RenderStats()
    keep, bgp = _bg(background)
    cam = camera._c()
    _check(_LIB.svlf_render_tiles_device(model.ctx.handle, model.handle, C.byref(cam), tile_w, tile_h, rank, world,
                                         bgp, _PREC[precision], C.c_void_p(d_rgb), C.c_void_p(d_alpha),
                                         C.c_void_p(d_depth), C.byref(st)))
    _add_stats(stats, st)


def render_rays(model: Model, rays, stats: RenderStats | None = None, background=None, precision="fp32"):
    """render_ray per ray (render.hpp:75), batched: returns (rgb n x 3, alpha n, depth n)."""
    r = _f64(rays).reshape(-1, 6)
    n = r.shape[0]
    rgb = np.zeros(n * 3, np.float32)
    alpha = np.zeros(n, np.float32)
    depth = np.zeros(n, np.float32)
    st = _RenderStats()
    keep, bgp = _bg(background)
    _check(_LIB.svlf_render_rays(model.ctx.handle, model.handle, _dp(r), n, bgp, _PREC[precision], _dp(rgb),
                                 _dp(alpha), _dp(depth), C.byref(st)))
    _add_stats(stats, st)
    return rgb.reshape(n, 3), alpha, depth


def _add_stats(stats, st):
    if stats is not None:
        for f, _ in _RenderStats._fields_:
            setattr(stats, f, getattr(stats, f) + getattr(st, f))


def _batch(rays, c_gt, depth_gt, alpha_gt):
    r = _f64(rays).reshape(-1, 6)
    n = r.shape[0]
    c = _f32(c_gt).reshape(n * 3)
    d = _f64(depth_gt).reshape(n)
    a = np.asarray(alpha_gt).reshape(n)
    if a.dtype == np.bool_:
        a = a.view(np.uint8)
    if a.dtype != np.uint8 or not a.flags.c_contiguous:  # any nonzero = foreground (the library reads != 0)
        a = np.ascontiguousarray(a != 0, dtype=np.uint8)
    return r, c, d, a, n


def train_step(model: Model, rays, c_gt, depth_gt, alpha_gt, mode: str = "volumetric",
               color_frozen: bool = False, lr: float = 1e-3, weights: LossWeights | None = None,
               stats: LossStats | None = None) -> float:
    """One optimizer step over a ray batch (src/train.cpp:443-479). Returns the loss sum."""
    r, c, d, a, n = _batch(rays, c_gt, depth_gt, alpha_gt)
    lw = (weights or LossWeights())._c()
    st = _LossStats()
    loss = C.c_double()
    _check(_LIB.svlf_train_step(model.ctx.handle, model.handle, _dp(r), _dp(c), _dp(d), _dp(a), n,
                                0 if mode == "surface" else 1, int(color_frozen), C.c_float(lr), C.byref(lw),
                                C.byref(st), C.byref(loss)))
    _add_loss_stats(stats, st)
    return loss.value


def train_step_device(model: Model, d_rays: int, d_cgt: int, d_depth: int, d_alpha: int, n: int,
                      mode: str = "volumetric", color_frozen: bool = False, lr: float = 1e-3,
                      weights: LossWeights | None = None, stats: LossStats | None = None) -> float:
    """train_step with the batch resident in device memory (pointers as ints)."""
    lw = (weights or LossWeights())._c()
    st = _LossStats()
    loss = C.c_double()
    _check(_LIB.svlf_train_step_device(model.ctx.handle, model.handle, C.c_void_p(d_rays), C.c_void_p(d_cgt),
                                       C.c_void_p(d_depth), C.c_void_p(d_alpha), n, 0 if mode == "surface" else 1,
                                       int(color_frozen), C.c_float(lr), C.byref(lw), C.byref(st), C.byref(loss)))
    _add_loss_stats(stats, st)
    return loss.value


class TrainPipeline:
    """Pipelined optimizer steps over host batches (svlf_train_batch_stage /
    svlf_train_step_staged): stage() queues batch k + 1's upload (DMA from
    page-locked arrays, or page-locked staging filled by a background thread)
    while step() runs batch k. At most two batches are staged; each batch's
    arrays are kept (and must stay unchanged) until it has been stepped.

        pipe = TrainPipeline(model); pipe.stage(*batch[0])
        for k in range(K):
            if k + 1 < K: pipe.stage(*batch[k + 1])
            loss = pipe.step(lr=...)
    """

    def __init__(self, model: Model):
        self.model = model
        self._queue = []  # (slot, arrays) in staging order

    def stage(self, rays, c_gt, depth_gt, alpha_gt):
        r, c, d, a, n = _batch(rays, c_gt, depth_gt, alpha_gt)
        slot = C.c_int()
        _check(_LIB.svlf_train_batch_stage(self.model.ctx.handle, _dp(r), _dp(c), _dp(d), _dp(a), n,
                                           C.byref(slot)))
        self._queue.append((slot.value, (r, c, d, a)))

    def step(self, mode: str = "volumetric", color_frozen: bool = False, lr: float = 1e-3,
             weights: LossWeights | None = None, stats: LossStats | None = None) -> float:
        """train_step on the oldest staged batch; returns its loss sum."""
        if not self._queue:
            raise ValueError("no batch staged")
        slot, _arrays = self._queue.pop(0)
        lw = (weights or LossWeights())._c()
        st = _LossStats()
        loss = C.c_double()
        _check(_LIB.svlf_train_step_staged(self.model.ctx.handle, self.model.handle, slot,
                                           0 if mode == "surface" else 1, int(color_frozen), C.c_float(lr),
                                           C.byref(lw), C.byref(st), C.byref(loss)))
        _add_loss_stats(stats, st)
        return loss.value

    def drain(self):
        """Drops the staged batches that were not stepped."""
        while self._queue:
            slot, _arrays = self._queue.pop(0)
            _check(_LIB.svlf_train_batch_discard(self.model.ctx.handle, slot))

    def __len__(self):
        return len(self._queue)


def loss_grads(model: Model, rays, c_gt, depth_gt, alpha_gt, mode: str = "volumetric",
               color_frozen: bool = False, weights: LossWeights | None = None,
               stats: LossStats | None = None) -> float:
    """Loss sum and summed gradients (read with model.get_grads()), no optimizer step."""
    r, c, d, a, n = _batch(rays, c_gt, depth_gt, alpha_gt)
    lw = (weights or LossWeights())._c()
    st = _LossStats()
    loss = C.c_double()
    _check(_LIB.svlf_loss_grads(model.ctx.handle, model.handle, _dp(r), _dp(c), _dp(d), _dp(a), n,
                                0 if mode == "surface" else 1, int(color_frozen), C.byref(lw), C.byref(st),
                                C.byref(loss)))
    _add_loss_stats(stats, st)
    return loss.value


def _add_loss_stats(stats, st):
    if stats is not None:
        for f, _ in _LossStats._fields_:
            setattr(stats, f, getattr(stats, f) + getattr(st, f))
