"""Build libflashoverlap.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Sources: csrc/*.cpp (host plan, tuner, C ABI), csrc/runtime.cu (NCCL +
streams), csrc/kernels/*.cu (tcgen05 GEMM, post-reorder).  cudart is linked
statically; NCCL is the venv's 2.28.9 (the same libnccl.so.2 torch loads),
found through an rpath.  The library loads on a GPU-less host (no libcuda
link: driver entry points are fetched at run time).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libflashoverlap.so")
BUILD = os.path.join(ROOT, "build", "obj")

SOURCES = [
    "api_plan.cpp",
    "plan.cpp",
    "tuner.cpp",
    "runtime.cu",
    "loopback.cu",
    "emulated.cu",
    "kernels/gemm_tcgen05.cu",
    "kernels/post_reorder.cu",
]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError(f"NCCL headers not found under {base}")
    return inc, lib


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def _headers():
    hs = [os.path.join(ROOT, "include", "flashoverlap.h")]
    for d, _, fs in os.walk(CSRC):
        hs += [os.path.join(d, f) for f in fs if f.endswith((".h", ".cuh"))]
    return hs


def up_to_date() -> bool:
    """The in-tree library is newer than every source and header (object files
    are not needed: build/ does not travel to the GPU boxes)."""
    if not os.path.exists(OUT):
        return False
    newest = max([os.path.getmtime(h) for h in _headers()] +
                 [os.path.getmtime(os.path.join(CSRC, s)) for s in SOURCES])
    return os.path.getmtime(OUT) >= newest


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    inc, lib = nccl_dirs()
    os.makedirs(BUILD, exist_ok=True)
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-Wall",
              f"-I{os.path.join(ROOT, 'include')}", f"-I{inc}", "--expt-relaxed-constexpr",
              "-Xptxas", "-v"] + ARCH
    jobs, objs = [], []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src.replace("/", "_") + ".o")
        objs.append(obj)
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(path), hdr_mtime)):
            continue
        lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
        jobs.append(([nvcc()] + lang + common + ["-c", path, "-o", obj], src))

    def run(job):
        cmd, src = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return src, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for src, log in ex.map(run, jobs):
            if verbose and log:
                print(f"--- {src}\n{log}", file=sys.stderr)
    if jobs or force or not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        link = [nvcc(), "-shared", "-o", OUT] + objs + ARCH + [
            "-cudart", "static", f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker=-rpath,{lib}",
            "-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
