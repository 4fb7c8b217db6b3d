"""Build libfj.so for sm_100a with nvcc (in-tree, so it travels with gpurun)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Build libfj.so (or a diagnostic variant at `out` with extra -D defines)."""
    out = out or os.path.join(HERE, "libfj.so")
    objdir = os.path.join(HERE, "csrc") if not defines else os.path.dirname(out)
    srcs = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
    deps = srcs + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "fj.h")]
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in deps):
            return out
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    dflags = [f"-D{d}" for d in defines]
    procs = [subprocess.Popen([NVCC, *FLAGS, *dflags, "-c", s, "-o", o], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for s, o in zip(srcs, objs)]
    logs = []
    for src, pr in zip(srcs, procs):
        txt = pr.communicate()[0]
        logs.append(txt)
        if pr.returncode != 0:
            sys.stderr.write(txt)
            raise RuntimeError("nvcc failed on " + src)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
