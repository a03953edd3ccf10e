"""Build the in-tree sm_100a shared library ``_xmhd_b200.so`` with nvcc.

The .so is the C-ABI declared in ``include/xmhd_b200.h``.  It is built in-tree
(git-ignored) so that it travels with the repo snapshot to the GPU box.
"""

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(REPO, "include")
SO_NAME = "_xmhd_b200.so"
SO_PATH = os.path.join(PKG, SO_NAME)

SOURCES = ["stencil.cu", "vec.cu", "capi.cu", "divdiff.cpp", "steps.cpp", "hostio.cpp"]
HEADERS = ["common.cuh", "kernels.h"]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    # the bitwise contract: no FMA contraction in device or host code
    "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    "-shared",
    "-cudart", "static",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale():
    if not os.path.exists(SO_PATH):
        return True
    t = os.path.getmtime(SO_PATH)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(INCLUDE, "xmhd_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_so(force=False, verbose=False, extra=(), out=None):
    """Compile the C-ABI library if any source is newer than the .so.

    Each source compiles to an object in parallel (the translation units only
    share host-linkage launch functions), then nvcc links the shared library."""
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    out = out or SO_PATH
    if not force and out == SO_PATH and not _stale():
        return out
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "static")]
    tmp = tempfile.mkdtemp(prefix="xmhd_build_")

    def compile_one(src):
        obj = os.path.join(tmp, os.path.basename(src) + ".o")
        cmd = [nvcc()] + compile_flags + list(extra) + ["-I", INCLUDE, "-I", CSRC, "-c",
                                                        os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        results = list(pool.map(compile_one, SOURCES))
    for _, res in results:
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed building %s" % SO_NAME)
        if verbose and (res.stdout or res.stderr):
            print(res.stdout + res.stderr)
    link = [nvcc(), "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
            "-Xcompiler", "-fPIC", "-o", out] + [obj for obj, _ in results]
    if verbose:
        print(" ".join(link), flush=True)
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking %s" % SO_NAME)
    for obj, _ in results:
        os.remove(obj)
    os.rmdir(tmp)
    return out


if __name__ == "__main__":
    build_so(force="--force" in sys.argv, verbose=True,
             extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else [])
