"""Build libreusevit.so in-tree with nvcc for sm_100a (no torch extension: the ABI is plain C).

    python -m paper_2506_14107_b200.build        (or __graft_entry__.build())
Objects are compiled in parallel; the shared library links the CUDA runtime statically so the
library does not depend on which libcudart the Python process has loaded.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(OUT_DIR, "libreusevit.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-I" + os.path.join(os.path.dirname(HERE), "include")]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(os.path.join(OUT_DIR, "obj"), exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers += [os.path.join(os.path.dirname(HERE), "include", f)
                for f in os.listdir(os.path.join(os.path.dirname(HERE), "include"))]
    objs, jobs = [], []
    for src in sources():
        obj = os.path.join(OUT_DIR, "obj", os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)
        return cmd[-1]

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if jobs or not os.path.exists(LIB):
        run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"])
    return LIB


def build_variant(out_path: str, defines=()) -> str:
    """Experiment builds (e.g. -DRV_ATTN_TRACE): all sources with extra -D flags into out_path;
    load with _lib.load_library(out_path) before the first ReuseViT.  Never the product library."""
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    objs = []
    for src in sources():
        obj = out_path + "." + os.path.basename(src) + ".o"
        subprocess.run([NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj], check=True)
        objs.append(obj)
    subprocess.run([NVCC, *ARCH, "-shared", "-o", out_path, *objs, "-cudart", "static"], check=True)
    return out_path


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
