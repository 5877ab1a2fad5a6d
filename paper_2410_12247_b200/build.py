"""Build the in-tree shared libraries with nvcc for sm_100a (no JIT cache).

  paper_2410_12247_b200/libepsmoe.so   the layer (C ABI of include/epsmoe.h)
  gen/libepsgen.so                      the device twin of the input generator

Usage: python -m paper_2410_12247_b200.build   (or __graft_entry__.build()).
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def nccl_paths():
    import nvidia.nccl  # torch's bundled NCCL (2.28.x): headers + libnccl.so.2
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False) -> list:
    nvcc = _nvcc()
    inc, lib = nccl_paths()
    built = []
    csrc = os.path.join(PKG, "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cpp")))
    deps = srcs + glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh")) + \
        [os.path.join(ROOT, "include", "epsmoe.h")]
    out = os.path.join(PKG, "libepsmoe.so")
    if force or _stale(out, deps):
        cmd = [nvcc, *ARCH, *FLAGS, "-I", inc, "-I", os.path.join(ROOT, "include"), *srcs,
               "-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath,{lib}", "-o", out + ".tmp"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = _run(cmd)
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(out + ".tmp", out)
        built.append(out)
    gsrc = os.path.join(ROOT, "gen", "gen.cu")
    gout = os.path.join(ROOT, "gen", "libepsgen.so")
    if force or _stale(gout, [gsrc]):
        _run([nvcc, *ARCH, *FLAGS, gsrc, "-o", gout + ".tmp"])
        os.replace(gout + ".tmp", gout)
        built.append(gout)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
