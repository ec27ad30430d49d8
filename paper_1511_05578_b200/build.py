"""Build libscurve_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1511_05578_b200.build        (or __graft_entry__.build())

Compiles every csrc/*.cu to an object (in parallel) and links one shared
library next to this file.  cudart is linked statically by nvcc; cuFFT is
linked from the CUDA toolkit with an rpath so the .so loads on the GPU box
(same image) without LD_LIBRARY_PATH.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libscurve_b200.so")
BUILD = os.path.join(HERE, "..", "build", "obj")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps_mtime():
    ts = [os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)]
    ts.append(os.path.getmtime(os.path.join(HERE, "..", "include", "scurve_b200.h")))
    ts.append(os.path.getmtime(__file__))
    return max(ts)


def _compile(src: str, verbose: bool, objdir: str = BUILD) -> str:
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Compile and link; `out`/`defines` build variants for A/B experiments."""
    global FLAGS
    if not force and out == OUT and os.path.exists(OUT) and os.path.getmtime(OUT) >= _deps_mtime():
        return OUT
    FLAGS = FLAGS + [f"-D{d}" for d in defines]
    # variant builds (other `out`) get their own object directory, so several
    # can be built at once
    objdir = BUILD if out == OUT else os.path.join(BUILD, "var_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, objdir), srcs))
    tmp = out + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, f"-L{CUDA}/lib64", "-lcufft",
           "-Xlinker", f"-rpath={CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="-v" in sys.argv,
                out=outs[0] if outs else OUT, defines=defs))
