"""Build the C-ABI shared library in-tree (sm_100a only).

    python -m paper_1608_02148_b200.build        (or __graft_entry__.build())

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, one object per
translation unit (parallel), linked against the NCCL that torch ships
(nvidia/nccl in site-packages) so only one libnccl lives in the process.
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "librsvd_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        cand = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("NCCL headers (nvidia/nccl) not found")


def _flags():
    nr = nccl_root()
    return nr, ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(nr, "include")] + ARCH


HASH_FILE = os.path.join(OUT_DIR, "build.sha256")


def _content_hash(deps, flags):
    """sha256 over every source / header, this script and the compiler flags:
    the library is rebuilt whenever its inputs change (not by mtime, which a
    copied tree -- e.g. the GPU box's snapshot -- does not preserve)."""
    import hashlib
    h = hashlib.sha256()
    for d in sorted(deps):
        h.update(os.path.relpath(d, ROOT).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join(flags).encode())
    return h.hexdigest()


def build(force=False, verbose=False):
    nr, flags = _flags()
    os.makedirs(os.path.join(OUT_DIR, "obj"), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "rsvd_b200.h"), __file__]
    digest = _content_hash(deps, flags)
    if not force and os.path.exists(LIB) and os.path.exists(HASH_FILE) and open(HASH_FILE).read().strip() == digest:
        return LIB

    def compile_one(src):
        obj = os.path.join(OUT_DIR, "obj", os.path.basename(src) + ".o")
        cmd = [NVCC, "-c", src, "-o", obj] + flags
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s" % (src, r.stderr[-6000:]))
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(compile_one, srcs))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    libdir = os.path.join(nr, "lib")
    cmd = [NVCC, "-shared", "-o", LIB] + objs + ARCH + [
        "-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir, "-lcudart", "-lcuda",
        "-Xlinker", "--no-undefined"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    with open(HASH_FILE, "w") as f:
        f.write(digest + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
