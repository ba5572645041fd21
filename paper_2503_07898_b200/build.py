"""Build the in-tree CUDA library ``_lib/libvoxl_b200.so`` for sm_100a.

Every translation unit is compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into one
shared object. The .so stays in-tree (git-ignored, shipped to the GPU box by
gpurun) so the driver can see it loaded.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
OBJDIR = os.path.join(PKG, "_lib", "obj")
LIB = os.path.join(LIBDIR, "libvoxl_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    "-I" + os.path.join(PKG, "..", "include"),
]

SOURCES = ["grid.cpp", "sparse_grid.cpp", "multires_grid.cpp", "dense.cu", "sparse.cu", "multires.cu", "capi.cu"]


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJDIR, src + ".o")
    path = os.path.join(CSRC, src)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(PKG, "..", "include", "voxl_b200.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [NVCC] + FLAGS + ["-x", "cu", "-c", path, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


CLI = os.path.join(LIBDIR, "voxl_b200")


def _json_include() -> str:
    """nlohmann/json (3.11, header-only) as vendored by the image's cudnn
    frontend -- the JSON library the reference's config parser uses."""
    import site

    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        d = os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.exists(os.path.join(d, "json.hpp")):
            return d
    raise RuntimeError("nlohmann/json.hpp not found (cudnn_frontend thirdparty headers)")


def build_cli() -> str:
    """The C++ driver (csrc/cli/voxl_b200_main.cpp): `voxl_b200 run|verify`,
    linked against the in-tree library with an $ORIGIN rpath."""
    src = os.path.join(CSRC, "cli", "voxl_b200_main.cpp")
    hdr = os.path.join(PKG, "..", "include", "voxl_b200.hpp")
    if os.path.exists(CLI) and os.path.getmtime(CLI) >= max(os.path.getmtime(x) for x in (src, hdr, LIB)):
        return CLI
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I" + os.path.join(PKG, "..", "include"), "-I" + _json_include(),
           src, "-L" + LIBDIR, "-lvoxl_b200", "-Wl,-rpath,$ORIGIN", "-o", CLI]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"voxl_b200 CLI build failed:\n{r.stderr}")
    return CLI


def build(verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-lcuda", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    build_cli()
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
