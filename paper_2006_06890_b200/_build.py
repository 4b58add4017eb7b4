"""In-tree build of the native library (libzcgraph_b200.so) for sm_100a.

nvcc cross-compiles without a GPU, so this runs in the build container and
the resulting .so travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_NAME = "libzcgraph_b200.so"
LIB_PATH = os.path.join(PKG, LIB_NAME)
# measurement probes (include/zcprobe.h): a separate tool library linked
# against the product library, so the traversal ABI exports no probe symbols
PROBE_LIB_NAME = "libzcprobe_b200.so"
PROBE_LIB_PATH = os.path.join(PKG, PROBE_LIB_NAME)

SOURCES = ["zc_api.cu", "zc_kernels.cu", "zc_gen.cu", "zc_compress.cu"]
PROBE_SOURCES = ["zc_probe.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build the zcgraph CUDA library")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> str:
    """Compile every .cu under csrc/ into the in-tree shared libraries (the
    product library and the probe tool library)."""
    _build_lib(SOURCES, LIB_PATH, [], force, verbose)
    _build_lib(PROBE_SOURCES, PROBE_LIB_PATH,
               ["-L", PKG, "-l:" + LIB_NAME, "-Xlinker", "-rpath,$ORIGIN"], force, verbose,
               extra_deps=[LIB_PATH])
    return LIB_PATH


def _build_lib(sources, lib_path, link_extra, force, verbose, extra_deps=()):
    srcs = [os.path.join(CSRC, s) for s in sources]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps += [os.path.join(ROOT, "include", f) for f in ("zcgraph.h", "zcprobe.h")]
    deps += list(extra_deps)
    if not force and not _stale(lib_path, deps):
        return lib_path
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    headers = [d for d in deps if d.endswith((".cuh", ".h"))]
    jobs = []
    objs = []
    for src in srcs:  # compile the translation units in parallel, stale ones only
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [src] + headers):
            continue
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", src,
               "-o", obj]
        jobs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                stderr=subprocess.PIPE, text=True)))
    for src, obj, proc in jobs:
        _, err = proc.communicate()
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{err}")
        if verbose:
            print(err)
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(err)
    tmp = lib_path + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, *link_extra, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    print(build_native(force=True, verbose=False))
