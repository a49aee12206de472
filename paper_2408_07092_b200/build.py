"""Build libds.so in-tree: nvcc -gencode arch=compute_100a,code=sm_100a.

Run as ``python -m paper_2408_07092_b200.build`` or through
``__graft_entry__.build()``.  Objects are compiled in parallel into
``build/``; the shared library lands next to this file so it travels to
the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "libds")
LIB = os.path.join(PKG, "libds.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "ds.h")]


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    newest = max(os.path.getmtime(d) for d in _deps())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj, ""
    p = subprocess.run([NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj], capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr}")
    return obj, p.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, _sources()))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs])
        os.replace(tmp, LIB)
    return LIB


def build_trace() -> str:
    """Debug library with per-CTA phase timestamps (-DDS_TRACE), one unity TU."""
    os.makedirs(BUILD, exist_ok=True)
    unity = os.path.join(BUILD, "unity_trace.cu")
    with open(unity, "w") as f:
        for src in _sources():
            f.write('#include "%s"\n' % src)
    # DS_TRACE_FLAGS / DS_TRACE_NAME: extra -D switches of timing experiments
    out = os.path.join(PKG, os.environ.get("DS_TRACE_NAME", "libds_trace.so"))
    extra = os.environ.get("DS_TRACE_FLAGS", "").split()
    subprocess.check_call([NVCC, *ARCH, *[x for x in FLAGS if x not in ("-v", "-Xptxas")], "-DDS_TRACE", *extra,
                           "-shared", unity, "-o", out])
    return out


def build_exp(name: str, flags: list[str]) -> str:
    """Timing-experiment variant of the product library (unity TU, extra -D switches)."""
    os.makedirs(BUILD, exist_ok=True)
    unity = os.path.join(BUILD, "unity_%s.cu" % name)
    with open(unity, "w") as f:
        for src in _sources():
            f.write('#include "%s"\n' % src)
    out = os.path.join(PKG, name + ".so")
    subprocess.check_call([NVCC, *ARCH, *[x for x in FLAGS if x not in ("-v", "-Xptxas")], *flags,
                           "-shared", unity, "-o", out])
    return out


if __name__ == "__main__":
    if "--trace" in sys.argv:
        print(build_trace())
    elif "--exp" in sys.argv:  # --exp NAME -DFLAG ...
        i = sys.argv.index("--exp")
        print(build_exp(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        print(build(verbose="-v" in sys.argv))
