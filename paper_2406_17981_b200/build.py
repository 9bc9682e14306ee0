"""In-tree build of libtoesplit.so.1 for sm_100a (nvcc cross-compiles without
a GPU). Objects go to paper_2406_17981_b200/build/, the shared library (plus
the libtoesplit.so symlink) next to this file so it travels with gpurun.

    python paper_2406_17981_b200/build.py [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libtoesplit.so.1")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
                   "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills", "-I", INC, "-I", CSRC]
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-Wall", "-Wno-unused-function",
             "-I", INC, "-I", CSRC, "-I", "/usr/local/cuda/include"]


def _sources():
    out = []
    for f in sorted(os.listdir(CSRC)):
        if f.endswith(".cu") or f.endswith(".cpp"):
            out.append(os.path.join(CSRC, f))
    return out


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    hs += [os.path.join(INC, f) for f in os.listdir(INC) if f.endswith(".h")]
    return hs


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def _compile(src: str, force: bool, obj_dir: str = OBJ, extra=()) -> str:
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
            os.path.getmtime(src), _newest(_headers())):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + CU_FLAGS + list(extra) + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXX_FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, variant: str = "", extra=()) -> str:
    """variant: name of an A/B build (objects in build/<variant>/, library
    ab/libtoesplit_<variant>.so, compiled with the extra nvcc flags)."""
    obj_dir = os.path.join(OBJ, variant) if variant else OBJ
    lib = os.path.join(ROOT, "ab", f"libtoesplit_{variant}.so") if variant else LIB
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, obj_dir, extra), srcs))
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < _newest(objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + [
            "-Xlinker", "-soname=libtoesplit.so.1", "-Xlinker", "-Bsymbolic",
            "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map"),
            "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if variant:
        return lib
    link = os.path.join(HERE, "libtoesplit.so")
    if os.path.islink(link) or os.path.exists(link):
        os.remove(link)
    os.symlink("libtoesplit.so.1", link)
    return LIB


if __name__ == "__main__":
    # python build.py [--force] [--variant NAME -DFLAG ...]
    args = sys.argv[1:]
    if "--variant" in args:
        i = args.index("--variant")
        print(build(force="--force" in args, variant=args[i + 1],
                    extra=[a for a in args[i + 2:] if a != "--force"]))
    else:
        print(build(force="--force" in args))
