"""Build libsand.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsand.so")
SOURCES = ["sand_api.cu", "lookup.cu", "tmlp_simt.cu", "tmlp_tc.cu", "tmlp_tc2.cu", "tmlp_tc3.cu", "tmlp_tc4.cu", "tmlp_x3.cu", "depthpop.cu", "mesh.cu"]
HEADERS = ["ptx.cuh", "sand_internal.h", "tmlp_common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# extra defines for diagnostic builds, e.g. SAND_BUILD_DEFS="-DSAND_HANG_DEBUG" (bounded mbarrier waits)
EXTRA = os.environ.get("SAND_BUILD_DEFS", "").split()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]


STAMP = LIB + ".flags"


def _flag_line():
    # path-independent (the repo is copied elsewhere on the GPU box): the include dir is written relatively
    return " ".join(["nvcc", *FLAGS, *EXTRA]).replace(ROOT, "<repo>")


def _stale():
    """Rebuild when the .so is missing, older than a source, or built with other flags / defines (a
    diagnostic SAND_BUILD_DEFS build is never silently reused by a default build, and vice versa)."""
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    if open(STAMP).read().strip() != _flag_line():
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "sand.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=True, ptxas_v=False):
    if not force and not _stale():
        return LIB
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *EXTRA, "-c", os.path.join(CSRC, src), "-o", obj]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    ok = True
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0 or (verbose and out.strip()):
            sys.stderr.write(f"[nvcc {src}]\n{out}\n")
        ok &= p.returncode == 0
    if not ok:
        raise RuntimeError("nvcc failed")
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
                           "-cudart", "static"])
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(_flag_line() + "\n")
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, ptxas_v="-v" in sys.argv)
    print(LIB)
