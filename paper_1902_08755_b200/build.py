"""Build libeqc.so (the C-ABI library) for sm_100a with nvcc, in-tree.

    python -m paper_1902_08755_b200.build [--force]

Compiles every .cu under csrc/ with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` into
``paper_1902_08755_b200/libeqc.so`` (static CUDA runtime; NCCL linked from the
torch-bundled ``nvidia/nccl`` wheel with an rpath to it).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libeqc.so")
OBJ = os.path.join(HERE, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nccl_dirs():
    """(include dir, lib dir) of the NCCL that torch loads (site-packages nvidia/nccl)."""
    cands = [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")]
    try:
        import nvidia  # type: ignore
        for p in getattr(nvidia, "__path__", []):
            cands.append(os.path.join(p, "nccl"))
    except Exception:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return None, None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=(), extra=()) -> str:
    """Compile and link libeqc.  ``out``/``defines`` build tuning variants
    (e.g. ``defines=["EQC_ENC_WARPS=4"]``) next to the default library."""
    if out == LIB and not defines and not extra and not force and not needs_build():
        return LIB
    obj_dir = OBJ if out == LIB else out + ".objs"
    os.makedirs(obj_dir, exist_ok=True)
    inc, libdir = nccl_dirs()
    extra_inc = ["-I", INCLUDE] + (["-I", inc] if inc else [])
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *CFLAGS, *extra, *extra_inc, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if inc:
            cmd += ["-DEQC_HAVE_NCCL=1"]
        if verbose:
            print(" ".join(cmd))
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), src))
        objs.append(obj)
    failed = []
    for pr, src in procs:
        log, _ = pr.communicate()
        if log and (verbose or pr.returncode):
            sys.stderr.write(log.decode(errors="replace"))
        if pr.returncode:
            failed.append(src)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    link = [NVCC, *ARCH, "-shared", "-o", out + ".tmp", *objs, "-cudart", "static"]
    if libdir:
        link += ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}"]
    if verbose:
        print(" ".join(link))
    subprocess.check_call(link)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
