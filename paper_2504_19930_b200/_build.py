"""Build the sm_100a C-ABI library in-tree (nvcc, no torch linkage).

Produces ``paper_2504_19930_b200/_lib/libechoreg_sm100.so`` from
``csrc/*.cu``.  Called by ``__graft_entry__.build()``; nvcc cross-compiles
without a GPU.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIB = os.path.join(LIBDIR, "libechoreg_sm100.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                "-Xptxas", "-v", "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]
# extra -D flags for kernel variant experiments (tools/), e.g. "-DER_OCT_PREFETCH=0"
FLAGS += os.environ.get("ER_NVCC_EXTRA", "").split()


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INCLUDE, "echoreg_b200.h"))
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src, obj, log):
    cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    sys.path.insert(0, CSRC)
    try:
        import gen_ziggurat
    finally:
        sys.path.pop(0)
    gen_ziggurat.main(os.path.join(CSRC, "zig_tables.h"))
    sources = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    hdrs = _headers()
    stamp = os.path.join(OBJDIR, "flags.stamp")
    if not os.path.exists(stamp) or open(stamp).read() != " ".join(FLAGS):
        for f in os.listdir(OBJDIR):
            if f.endswith(".o"):
                os.remove(os.path.join(OBJDIR, f))
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(sources), os.cpu_count() or 1))) as ex:
        for f in sources:
            src = os.path.join(CSRC, f)
            obj = os.path.join(OBJDIR, f[:-3] + ".o")
            if _stale(obj, [src, *hdrs]):
                jobs.append(ex.submit(_compile, src, obj, obj + ".log"))
        for j in jobs:
            j.result()
    objs = [os.path.join(OBJDIR, f[:-3] + ".o") for f in sources]
    stamp = os.path.join(OBJDIR, "flags.stamp")
    open(stamp, "w").write(" ".join(FLAGS))
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
