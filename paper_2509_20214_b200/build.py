"""Build libqpalette.so in-tree (nvcc for sm_100a, host C++17 via nvcc's host compiler).

    python -m paper_2509_20214_b200.build [--jobs N] [--force]

Objects go to paper_2509_20214_b200/build/; the shared library to
paper_2509_20214_b200/libqpalette.so (git-ignored, shipped to the GPU box by gpurun).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libqpalette.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    for base in sys.path + [sysconfig.get_paths()["purelib"]]:
        d = os.path.join(base, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return os.path.join(d, "include"), os.path.join(d, "lib")
    raise RuntimeError("NCCL headers not found (expected the nvidia-nccl wheel in site-packages)")


def _needs(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(jobs: int = 0, force: bool = False, verbose: bool = False, defines: list[str] | None = None,
          out: str | None = None) -> str:
    """defines / out: experimental variants (-D flags) built into a separate object dir and .so."""
    lib_path = out or LIB
    bdir = BUILD if not defines else BUILD + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(bdir, exist_ok=True)
    inc_nccl, lib_nccl = nccl_dirs()
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "qpalette.h")]
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    common = ["-std=c++17", "-O3", "-Xcompiler", "-fPIC", "-I", inc_nccl, "-I", CSRC,
              "-I", os.path.join(HERE, "..", "include")] + ["-D" + d for d in (defines or [])]
    cmds = []
    objs = []
    for s in srcs:
        obj = os.path.join(bdir, os.path.basename(s) + ".o")
        objs.append(obj)
        if force or _needs(obj, [s] + headers):
            if s.endswith(".cu"):
                cmd = ["nvcc", *ARCH, "-lineinfo", *common, "-c", s, "-o", obj]
            else:
                cmd = ["nvcc", "-x", "c++", *common, "-c", s, "-o", obj]
            cmds.append(cmd)
    jobs = jobs or os.cpu_count() or 4

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("compile failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose:
            print(" ".join(cmd[-3:]), flush=True)
        return r

    with cf.ThreadPoolExecutor(jobs) as ex:
        list(ex.map(run, cmds))
    if force or cmds or not os.path.exists(lib_path):
        link = ["nvcc", *ARCH, "-shared", "-o", lib_path, *objs, "-L", lib_nccl, "-l:libnccl.so.2",
                "-Xlinker", "-rpath," + lib_nccl, "-cudart", "static"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed: " + " ".join(link) + "\n" + r.stdout + r.stderr)
    return lib_path


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=0)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    print(build(a.jobs, a.force, verbose=True, defines=a.defines, out=a.out))
