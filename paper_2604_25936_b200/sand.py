"""ctypes binding of libsand (include/sand.h).  Argument marshalling only.

Every compute step of a query runs in libsand's CUDA kernels.  There is no CPU fallback: if the
shared library is missing or no B200 is present, the calls raise.  Torch is used by callers only to
own device memory and streams (pass ``tensor.data_ptr()`` / ``stream.cuda_stream``).
"""
import ctypes
import os

import numpy as np

from .build import LIB as _LIB_PATH

SAND_OK = 0
SAND_ERR_ARG, SAND_ERR_STATE, SAND_ERR_SIZE, SAND_ERR_DEPTHMAP = -1, -2, -3, -4
SAND_ERR_CUDA, SAND_ERR_OOM, SAND_ERR_UNSUPPORTED = -5, -6, -7
SAND_FP32, SAND_TF32X3, SAND_BF16, SAND_F16X3 = 0, 1, 2, 3
SAND_TAIL_LINEAR, SAND_TAIL_MULT = 0, 1
SAND_OPT_PAIR_KERNEL, SAND_OPT_DYN_SCHEDULE, SAND_OPT_KPROF, SAND_OPT_FP32_TENSOR = 1, 2, 3, 4
SAND_MAX_L = 32
SAND_DEPTH_NONFINITE = 255


class SandError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libsand error {code}: {msg}")
        self.code = code


class sand_config(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int), ("H", ctypes.c_int), ("omega0", ctypes.c_float),
                ("prec", ctypes.c_int), ("tail", ctypes.c_int), ("device", ctypes.c_int)]


class sand_depthmap(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("level", ctypes.c_int),
                ("depth", ctypes.POINTER(ctypes.c_uint8)), ("far_sdf", ctypes.POINTER(ctypes.c_float)),
                ("nodes", ctypes.POINTER(ctypes.c_uint32)),
                ("n_nodes", ctypes.c_int64), ("n_leaves", ctypes.c_int64)]


class sand_stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("n_nonfinite", ctypes.c_int64),
                ("per_depth", ctypes.c_int64 * (SAND_MAX_L + 1)), ("tiles", ctypes.c_int64),
                ("flops_exec", ctypes.c_double), ("flops_ns", ctypes.c_double),
                ("ms_lookup", ctypes.c_float), ("ms_bin", ctypes.c_float),
                ("ms_mlp", ctypes.c_float), ("ms_total", ctypes.c_float),
                ("queries", ctypes.c_int64), ("ms_lookup_sum", ctypes.c_double), ("ms_bin_sum", ctypes.c_double),
                ("ms_mlp_sum", ctypes.c_double), ("ms_total_sum", ctypes.c_double)]


EXPORTS = ("sand_create", "sand_destroy", "sand_load_weights", "sand_load_depthmap", "sand_set_stream",
           "sand_set_lod_cap", "sand_reserve", "sand_query", "sand_query_host", "sand_get_stats",
           "sand_debug_perm", "sand_last_error", "sand_abi_version", "sand_required_depth",
           "sand_populate_leaf_depths", "sand_query_dynamic", "sand_marching_cubes", "sand_mesh_grid",
           "sand_set_option", "sand_get_option")

_lib = None


def load_library(path=None):
    """Load libsand.so (built in-tree by build.py).  Raises if it is missing -- no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("SAND_LIB") or _LIB_PATH   # SAND_LIB: diagnostic A/B builds
    if not os.path.exists(path):
        raise ImportError(f"libsand.so not found at {path}; run `python -m paper_2604_25936_b200.build`")
    lib = ctypes.CDLL(path)
    vp, i64, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
    lib.sand_create.argtypes = [ctypes.POINTER(sand_config), ctypes.POINTER(vp)]
    lib.sand_destroy.argtypes = [vp]
    lib.sand_load_weights.argtypes = [vp, ctypes.POINTER(ctypes.c_float), sz]
    lib.sand_load_depthmap.argtypes = [vp, ctypes.POINTER(sand_depthmap)]
    lib.sand_set_stream.argtypes = [vp, vp]
    lib.sand_set_lod_cap.argtypes = [vp, ctypes.c_int]
    lib.sand_reserve.argtypes = [vp, i64]
    lib.sand_set_option.argtypes = [vp, ctypes.c_int, i64]
    lib.sand_get_option.argtypes = [vp, ctypes.c_int, ctypes.POINTER(i64)]
    lib.sand_query.argtypes = [vp, vp, i64, vp, vp]
    lib.sand_query_host.argtypes = [vp, vp, i64, vp, vp, i64]
    lib.sand_get_stats.argtypes = [vp, ctypes.POINTER(sand_stats)]
    lib.sand_debug_perm.argtypes = [vp, vp, i64, ctypes.POINTER(i64)]
    lib.sand_last_error.argtypes = [vp]
    lib.sand_last_error.restype = ctypes.c_char_p
    lib.sand_abi_version.argtypes = []
    lib.sand_required_depth.argtypes = [vp, vp, i64, ctypes.c_float, ctypes.c_int, vp]
    lib.sand_populate_leaf_depths.argtypes = [vp, vp, i64, ctypes.c_int, ctypes.c_float, vp]
    lib.sand_query_dynamic.argtypes = [vp, vp, i64, ctypes.c_float, vp, vp]
    lib.sand_marching_cubes.argtypes = [vp, vp, ctypes.c_int, vp, i64, ctypes.POINTER(i64)]
    lib.sand_mesh_grid.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, i64, ctypes.POINTER(i64)]
    for f in EXPORTS:
        if f not in ("sand_last_error",):
            getattr(lib, f).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(lib, ctx, rc):
    if rc != SAND_OK:
        raise SandError(rc, lib.sand_last_error(ctx).decode(errors="replace"))


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype)) if a is not None else None


class SandContext:
    """One libsand context (one device).  Thin wrapper over the C ABI; same call names."""

    def __init__(self, L, H, omega0=30.0, prec=SAND_BF16, tail=SAND_TAIL_LINEAR, device=0):
        self.lib = load_library()
        self.cfg = sand_config(L, H, float(omega0), prec, tail, device)
        h = ctypes.c_void_p()
        _check(self.lib, None, self.lib.sand_create(ctypes.byref(self.cfg), ctypes.byref(h)))
        self.h = h
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            self.lib.sand_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, rc):
        _check(self.lib, self.h, rc)

    # -- loaders ----------------------------------------------------------------------------------
    def sand_load_weights(self, blob):
        blob = np.ascontiguousarray(blob, np.float32)
        self._chk(self.lib.sand_load_weights(self.h, _ptr(blob, ctypes.c_float), blob.size))

    def sand_load_depthmap(self, dm):
        """dm: a sandgen VoxelMap / Octree (or any object with the same fields)."""
        if hasattr(dm, "nodes"):
            depth = np.ascontiguousarray(dm.leaf_depth, np.uint8)
            far = None if dm.leaf_far_sdf is None else np.ascontiguousarray(dm.leaf_far_sdf, np.float32)
            nodes = np.ascontiguousarray(dm.nodes, np.uint32)
            s = sand_depthmap(1, dm.level, _ptr(depth, ctypes.c_uint8), _ptr(far, ctypes.c_float),
                              _ptr(nodes, ctypes.c_uint32), nodes.size, depth.size)
        else:
            depth = np.ascontiguousarray(dm.depth, np.uint8)
            far = None if dm.far_sdf is None else np.ascontiguousarray(dm.far_sdf, np.float32)
            s = sand_depthmap(0, dm.level, _ptr(depth, ctypes.c_uint8), _ptr(far, ctypes.c_float), None, 0, 0)
        self._chk(self.lib.sand_load_depthmap(self.h, ctypes.byref(s)))

    def sand_set_stream(self, stream_ptr):
        self._chk(self.lib.sand_set_stream(self.h, ctypes.c_void_p(int(stream_ptr) if stream_ptr else 0)))

    def sand_set_lod_cap(self, cap):
        self._chk(self.lib.sand_set_lod_cap(self.h, int(cap)))

    def sand_set_option(self, option, value):
        self._chk(self.lib.sand_set_option(self.h, int(option), int(value)))

    def sand_get_option(self, option):
        v = ctypes.c_int64()
        self._chk(self.lib.sand_get_option(self.h, int(option), ctypes.byref(v)))
        return v.value

    def sand_reserve(self, n_max):
        self._chk(self.lib.sand_reserve(self.h, int(n_max)))

    # -- queries ----------------------------------------------------------------------------------
    def sand_query(self, d_points, n, d_sdf, d_depth):
        """Device pointers (ints, e.g. torch tensor .data_ptr())."""
        self._chk(self.lib.sand_query(self.h, ctypes.c_void_p(d_points), int(n), ctypes.c_void_p(d_sdf),
                                      ctypes.c_void_p(d_depth)))

    def sand_query_host(self, h_points, n, h_sdf, h_depth, chunk_points=0):
        """Host pointers (ints; pinned memory for full bandwidth)."""
        self._chk(self.lib.sand_query_host(self.h, ctypes.c_void_p(h_points), int(n), ctypes.c_void_p(h_sdf),
                                           ctypes.c_void_p(h_depth), int(chunk_points)))

    def sand_get_stats(self):
        s = sand_stats()
        self._chk(self.lib.sand_get_stats(self.h, ctypes.byref(s)))
        L = self.cfg.L
        return dict(n=s.n, n_nonfinite=s.n_nonfinite, per_depth=list(s.per_depth[:L + 1]), tiles=s.tiles,
                    flops_exec=s.flops_exec, flops_ns=s.flops_ns, ms_lookup=s.ms_lookup, ms_bin=s.ms_bin,
                    ms_mlp=s.ms_mlp, ms_total=s.ms_total, queries=s.queries, ms_lookup_sum=s.ms_lookup_sum,
                    ms_bin_sum=s.ms_bin_sum, ms_mlp_sum=s.ms_mlp_sum, ms_total_sum=s.ms_total_sum)

    def sand_debug_perm(self):
        nb = ctypes.c_int64()
        self._chk(self.lib.sand_debug_perm(self.h, None, 0, ctypes.byref(nb)))
        out = np.empty(nb.value, np.uint32)
        self._chk(self.lib.sand_debug_perm(self.h, out.ctypes.data_as(ctypes.c_void_p), out.size, ctypes.byref(nb)))
        return out

    # -- depth-map population (Eq. 5 / Eq. 6) --------------------------------------------------------
    def sand_required_depth(self, d_points, n, r, near, d_out_depth):
        self._chk(self.lib.sand_required_depth(self.h, ctypes.c_void_p(d_points), int(n), float(r), int(bool(near)),
                                               ctypes.c_void_p(d_out_depth)))

    def sand_populate_leaf_depths(self, d_samples, n_leaves, samples_per_leaf, r, d_leaf_depth):
        self._chk(self.lib.sand_populate_leaf_depths(self.h, ctypes.c_void_p(d_samples), int(n_leaves),
                                                     int(samples_per_leaf), float(r), ctypes.c_void_p(d_leaf_depth)))

    # -- dynamic exit without a depth map ('SAND w/o Octree') ----------------------------------
    def sand_query_dynamic(self, d_points, n, r, d_out_sdf, d_out_exit_depth):
        self._chk(self.lib.sand_query_dynamic(self.h, ctypes.c_void_p(d_points), int(n), float(r),
                                              ctypes.c_void_p(d_out_sdf), ctypes.c_void_p(d_out_exit_depth)))

    # -- marching cubes on the query grid ----------------------------------------------
    def sand_marching_cubes(self, d_sdf, R, d_tris, cap):
        n = ctypes.c_int64(0)
        self._chk(self.lib.sand_marching_cubes(self.h, ctypes.c_void_p(d_sdf), int(R), ctypes.c_void_p(d_tris),
                                               int(cap), ctypes.byref(n)))
        return n.value

    def sand_mesh_grid(self, R, slab, d_tris, cap):
        n = ctypes.c_int64(0)
        self._chk(self.lib.sand_mesh_grid(self.h, int(R), int(slab), ctypes.c_void_p(d_tris), int(cap),
                                          ctypes.byref(n)))
        return n.value

    # -- torch convenience (device tensors in, device tensors out) -----------------------------------
    def query_tensor(self, pts, sdf=None, depth=None):
        import torch
        assert pts.is_cuda and pts.dtype == torch.float32 and pts.is_contiguous() and pts.shape[-1] == 3
        n = pts.shape[0]
        if sdf is None:
            sdf = torch.empty(n, dtype=torch.float32, device=pts.device)
        if depth is None:
            depth = torch.empty(n, dtype=torch.uint8, device=pts.device)
        self.sand_set_stream(torch.cuda.current_stream(pts.device).cuda_stream)
        self.sand_query(pts.data_ptr(), n, sdf.data_ptr(), depth.data_ptr())
        return sdf, depth


def abi_version():
    return load_library().sand_abi_version()
