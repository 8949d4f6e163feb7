"""ctypes front end of the plain FP32 C oracle (oracle/sand_oracle_fp32.c).  TEST INFRASTRUCTURE ONLY.

``build()`` compiles it with gcc (-O2 -ffp-contract=off -fopenmp: IEEE binary32, no FMA contraction,
sequential sums, glibc sinf) into oracle/liboracle_fp32.so; ``query_fp32`` evaluates SAND's adaptive
query (Sec. 3.4, Eq. 2/3/7) on host cores.  Parameters and depth maps are passed duck-typed
like the float64 oracle (oracle/sand_oracle.py): this module imports nothing from the product package.
"""
import ctypes
import os
import platform
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sand_oracle_fp32.c")
LIB = os.path.join(HERE, "liboracle_fp32.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC", "-std=c11"]
_lib = None


def _compiler():
    # the system gcc ships libgomp (an alternative gcc earlier on PATH / in $CC may not)
    for cc in ("/usr/bin/gcc", os.environ.get("CC"), "gcc"):
        if cc and (os.path.sep not in cc or os.path.exists(cc)):
            return cc
    return "gcc"


def build(force=False):
    """Compile the C oracle if its .so is missing or older than the source."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    tmp = LIB + ".tmp"
    subprocess.check_call([_compiler(), *CFLAGS, SRC, "-o", tmp, "-lm"])
    os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        lib.oracle_query_fp32.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_float, ctypes.c_int,
                                          vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int,
                                          vp, vp, vp, ctypes.c_int, vp, i64, vp, vp, ctypes.c_int]
        lib.oracle_query_fp32.restype = ctypes.c_int
        lib.oracle_lookup_fp32.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int, vp, i64, vp, ctypes.c_int]
        lib.oracle_lookup_fp32.restype = ctypes.c_int
        lib.oracle_threads.argtypes = [ctypes.c_int]
        lib.oracle_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, np.float32))


def _ptr(a):
    return None if a is None else a.ctypes.data


def threads(nthreads=0):
    """OpenMP threads the oracle runs on (nthreads <= 0: the runtime default = usable cores)."""
    return int(_load().oracle_threads(int(nthreads)))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _map(depthmap):
    if hasattr(depthmap, "nodes"):
        return (1, np.ascontiguousarray(np.asarray(depthmap.nodes, np.uint32)),
                np.ascontiguousarray(np.asarray(depthmap.leaf_depth, np.uint8)), depthmap.leaf_far_sdf)
    return 0, None, np.ascontiguousarray(np.asarray(depthmap.depth, np.uint8)), depthmap.far_sdf


def lookup_fp32(depthmap, points, lod_cap=None, nthreads=0):
    """Exit depths only (cell in float32, descent, LOD cap; 255 for non-finite points), u8 [n]."""
    lib = _load()
    kind, nodes, dep, _ = _map(depthmap)
    pts = _f32(points).reshape(-1, 3)
    out = np.empty(pts.shape[0], np.uint8)
    rc = lib.oracle_lookup_fp32(kind, int(depthmap.level), _ptr(dep), _ptr(nodes), int(lod_cap or 0), _ptr(pts),
                                pts.shape[0], _ptr(out), int(nthreads))
    if rc != 0:
        raise ValueError("octree deeper than its declared level")
    return out


def query_fp32(params, depthmap, points, lod_cap=None, nthreads=0):
    """FP32 adaptive query (Sec. 3.4): returns (sdf float32 [n], exit depth u8 [n]); non-finite points
    give (NaN, 255)."""
    lib = _load()
    spec = params.spec
    L, H = int(spec.L), int(spec.H)
    W1 = _f32(params.W[0]).reshape(H, 3)
    Wh = _f32(np.stack([np.asarray(params.W[i], np.float32) for i in range(1, L)])) if L > 1 else None
    b = _f32(np.stack([np.asarray(params.b[i], np.float32) for i in range(L)]))
    a = _f32(np.stack([np.asarray(params.a[i], np.float32) for i in range(L)]))
    c = _f32([params.c[i] for i in range(L)])
    mult = int(spec.tail) == 1 and L > 1
    a1 = _f32(np.stack([np.asarray(params.a1[i], np.float32) for i in range(L - 1)])) if mult else None
    c1 = _f32([params.c1[i] for i in range(L - 1)]) if mult else None
    kind, nodes, dep, far = _map(depthmap)
    far = _f32(far) if far is not None else None
    pts = _f32(points).reshape(-1, 3)
    n = pts.shape[0]
    sdf = np.empty(n, np.float32)
    ed = np.empty(n, np.uint8)
    rc = lib.oracle_query_fp32(L, H, float(spec.omega0), int(spec.tail), _ptr(W1), _ptr(Wh), _ptr(b), _ptr(a),
                               _ptr(c), _ptr(a1), _ptr(c1), kind, int(depthmap.level), _ptr(dep), _ptr(far),
                               _ptr(nodes), int(lod_cap or 0), _ptr(pts), n, _ptr(sdf), _ptr(ed), int(nthreads))
    if rc != 0:
        raise ValueError("octree deeper than its declared level")
    return sdf, ed
