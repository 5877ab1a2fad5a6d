"""Per-kernel counts of the SASS mnemonics that prove tcgen05 / TMEM / TMA use
(B200_PROFILING.md: tcgen05.mma -> UTC*MMA, tcgen05.ld/st -> LDTM/STTM, TMA ->
UTMALDG/UTMASTG/UBLKCP).  Runs on the built library here (no GPU):

    python tools/sass_counts.py paper_2410_12247_b200/libepsmoe.so > profiles/r02_sass_counts.md
"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

PAT = re.compile(r"\b(UTC[A-Z]*MMA[A-Z0-9_.]*|UTCBAR[A-Z0-9_.]*|UTMALDG[A-Z0-9_.]*|UTMASTG[A-Z0-9_.]*|"
                 r"UBLKCP[A-Z0-9_.]*|LDTM[A-Z0-9_.]*|STTM[A-Z0-9_.]*|UTMACCTL[A-Z0-9_.]*|HMMA[A-Z0-9_.]*)")


def main(path):
    sass = subprocess.run(["cuobjdump", "-sass", path], check=True, capture_output=True, text=True).stdout
    demangle = lambda s: subprocess.run(["c++filt", s], capture_output=True, text=True).stdout.strip()
    funcs = OrderedDict()
    cur = None
    for line in sass.splitlines():
        if "Function :" in line:
            cur = line.split("Function :")[1].strip()
            funcs[cur] = Counter()
        elif cur:
            for m in PAT.findall(line):
                funcs[cur][m.rstrip(".")] += 1
    print(f"# SASS mnemonic counts of `{path}` (cuobjdump -sass, sm_100a)\n")
    print("`gemm_kernel<EPI, CG, GATHER>`: EPI 0 = GateUp+SwiGLU, 1 = Down (bf16), 2 = router (fp32), 3 = shared Down + "
          "combine; CG 2 = CTA pair (cta_group::2). Counts are static instruction sites, not executions.\n")
    print("| kernel | mnemonics |\n|---|---|")
    for f, c in funcs.items():
        if not c:
            continue
        name = demangle(f)
        name = re.sub(r"epsmoe::\(anonymous namespace\)::", "", name)
        name = re.sub(r"\(CUtensorMap_st.*", "", name)
        print(f"| `{name[:120]}` | " + ", ".join(f"{k} {v}" for k, v in sorted(c.items())) + " |")
    plain = [demangle(f) for f, c in funcs.items() if not c]
    print(f"\n{len(plain)} other kernels (routing, permute, combine, LocalReduce, p2p) are CUDA-core / LSU code "
          "with none of these mnemonics.")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2410_12247_b200/libepsmoe.so")
