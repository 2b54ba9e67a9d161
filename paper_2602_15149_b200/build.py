"""Build libtlsph.so (sm_100a) in-tree with nvcc.

    python -m paper_2602_15149_b200.build [--force]

The shared object lands next to this file so it travels to the GPU box with
the repo snapshot.  No JIT cache, no torch extension machinery: the library
exposes a plain C ABI (include/tlsph.h) loaded with ctypes.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libtlsph.so")
SOURCES = ["plugin.cu", "neighbors.cu", "tiles.cu", "step.cu", "output.cu", "contact.cu"]
HEADERS = ["tl_common.cuh", "expr_vm.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-ftz=true",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _deps():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "tlsph.h"))
    return files


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def _compile(src, obj, defines=()):
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src),
           "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    return res.stderr


def build(force=False, verbose=False, defines=(), out=None):
    """Compile and link.  ``defines``/``out`` build tuning variants (e.g.
    TL_GATHER_B=2 into libtlsph_g2.so) without touching the default library."""
    lib = out or LIB
    if not force and not defines and not needs_build():
        return lib
    tag = "" if not defines else "_" + "_".join(d.replace("=", "") for d in defines)
    objdir = os.path.join(HERE, "_obj" + tag)
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]
    # without force, recompile only the objects older than their source or a header
    hdr = max(os.path.getmtime(f) for f in _deps() if not f.endswith(".cu"))
    todo = [(src, obj) for src, obj in zip(SOURCES, objs)
            if force or not os.path.exists(obj)
            or os.path.getmtime(obj) < max(hdr, os.path.getmtime(os.path.join(CSRC, src)))]
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        logs = list(ex.map(lambda a: _compile(a[0], a[1], defines), todo))
    if verbose:
        for log in logs:
            print(log, file=sys.stderr)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=outs[0] if outs else None))
