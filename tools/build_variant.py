"""Dev A/B helper: build libepsmoe.so from a git revision into tools/ab/lib_<name>.so
(loaded with EPSMOE_LIB=<path>), so two kernel versions run on the same GPU box.

  python tools/build_variant.py <rev> <name> [-DMACRO=V ...]   (rev "WORKTREE" = the working tree)
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_12247_b200.build import ARCH, FLAGS, _nvcc, nccl_paths  # noqa: E402


def main(rev, name, *defs):
    d = tempfile.mkdtemp()
    if rev == "WORKTREE":
        subprocess.run(f"cd {ROOT} && tar -c paper_2410_12247_b200/csrc include | tar -x -C {d}", shell=True, check=True)
    else:
        subprocess.run(f"git -C {ROOT} archive {rev} paper_2410_12247_b200/csrc include | tar -x -C {d}",
                       shell=True, check=True)
    inc, lib = nccl_paths()
    csrc = os.path.join(d, "paper_2410_12247_b200", "csrc")
    srcs = sorted(os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith((".cu", ".cpp")))
    out = os.path.join(ROOT, "tools", "ab", f"lib_{name}.so")
    subprocess.run([_nvcc(), *ARCH, *FLAGS, *defs, "-I", inc, "-I", os.path.join(d, "include"), *srcs, "-L", lib,
                    "-l:libnccl.so.2", f"-Xlinker=-rpath,{lib}", "-o", out], check=True)
    print(out)


if __name__ == "__main__":
    main(*sys.argv[1:])
