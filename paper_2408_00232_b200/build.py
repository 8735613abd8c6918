"""Build libcdfgnn.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2408_00232_b200.build [--force] [--verbose]

Objects go to paper_2408_00232_b200/_build/, the library to
paper_2408_00232_b200/libcdfgnn.so (git-ignored; it travels to the GPU box
with the gpurun snapshot).  NCCL is the torch-bundled 2.28 (headers from the
nvidia-nccl wheel); the library links it by soname so the process shares the
copy torch already loaded.
"""
import argparse
import glob
import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libcdfgnn.so")
INCLUDE = os.path.join(ROOT, "include")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for base in spec.submodule_search_locations:
            cands.append(os.path.join(base, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + glob.glob(os.path.join(INCLUDE, "*.h")))


def _digest(src, cmd):
    """Content hash of a source, every header it may include and the compile command: an
    object is reused only when this matches its stamp (mtimes alone can be stale after a
    checkout or a copy)."""
    h = hashlib.sha256(" ".join(cmd).encode())
    for f in [src] + sorted(_headers()):
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def _compile(src, nccl_inc, force, verbose):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    stamp = obj + ".sha256"
    cmd = [NVCC, "-c", src, "-o", obj, "-O3", "-std=c++17", "-lineinfo", *ARCH,
           "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-I", INCLUDE, "-I", CSRC, "-I", nccl_inc,
           "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3"]
    dig = _digest(src, cmd)
    if not force and os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == dig:
        return obj, False
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    with open(stamp, "w") as fh:
        fh.write(dig)
    return obj, True


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        res = list(ex.map(lambda s: _compile(s, nccl_inc, force, verbose), srcs))
    objs = [o for o, _ in res]
    # stale objects of removed sources must not be linked
    for o in glob.glob(os.path.join(OBJ, "*.o")):
        if o not in objs:
            os.remove(o)
    if not force and not any(rebuilt for _, rebuilt in res) and os.path.exists(LIB) and \
            os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-shared", *ARCH, "-o", tmp, *objs, "-L", nccl_lib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + nccl_lib, "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
