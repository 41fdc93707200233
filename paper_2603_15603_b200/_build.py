"""Build recipe of the CUDA library (in-tree, sm_100a only).

    python -m paper_2603_15603_b200._build        # incremental
    python -m paper_2603_15603_b200._build --force

Compiles every csrc/*.cu with nvcc for sm_100a (-gencode
arch=compute_100a,code=sm_100a -lineinfo) in parallel and links
paper_2603_15603_b200/lib/libfsb_b200.so.  The .so is git-ignored but travels
to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.environ.get("FSB_OBJ_DIR") or os.path.join(ROOT, "build", "obj")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.environ.get("FSB_LIB_OUT") or os.path.join(LIB_DIR, "libfsb_b200.so")  # A/B variants: FSB_LIB_OUT
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include")]
if os.environ.get("FSB_PROFILE"):  # cycle-attribution counters in the tcgen05 kernels
    FLAGS.append("-DFSB_PROFILE")
if os.environ.get("FSB_EXTRA_FLAGS"):  # experiments: extra -D flags
    FLAGS.extend(os.environ["FSB_EXTRA_FLAGS"].split())
if os.environ.get("FSB_HANG_DEBUG"):  # mbarrier waits time out and report instead of hanging
    FLAGS.append("-DFSB_HANG_DEBUG")


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "fsb_b200.h"))
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose):
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed on %s:\n%s%s" % (src, r.stdout, r.stderr))
    return obj, r.stderr


def build(force=False, verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    srcs = _sources()
    hdrs = _headers()
    todo = [s for s in srcs
            if force or _stale(os.path.join(OBJ, os.path.basename(s)[:-3] + ".o"), [s, *hdrs])]
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(todo)))) as ex:
        for obj, log in ex.map(lambda s: _compile(s, verbose), todo):
            logs.append(log)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in srcs]
    if force or todo or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s%s" % (r.stdout, r.stderr))
    return LIB, "".join(logs)


if __name__ == "__main__":
    lib, log = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    if log.strip():
        print(log)
    print(lib)
