"""Summarise an ncu source-page CSV (SASS view) of gemm_kernel: for every
mbarrier try-wait site, its first-try executions, retry-loop executions and
stall samples, labelled by the SmemTail barrier it polls (offset from the
tail base).  Usage: python tools/ncu_waits.py <source.csv> [stages]"""
import csv
import re
import sys


def main(path, stages=6):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iSrc = hdr.index("Source")
    iE = hdr.index("Instructions Executed")
    iA = hdr.index("Address")
    base = 0x30000 if stages == 6 else None
    names = {}
    off = 0
    for nm, n in (("full", stages), ("empty", stages), ("tfull", 2), ("tempty", 2), ("gfull", stages), ("qfull", 4),
                  ("qempty", 4)):
        for i in range(n):
            names[off + 8 * i] = nm
        off += 8 * n
    tot = sum(float(r[iS] or 0) for r in data)
    agg = {}
    for i, r in enumerate(data):
        m = re.search(r"TRYWAIT P\d, \[R\d+\+URZ(?:\+(0x[0-9a-f]+))?\]", r[iSrc])
        if not m:
            continue
        o = int(m.group(1), 16) if m.group(1) else 0
        nm = names.get(o - base, hex(o)) if o >= base else hex(o)
        e = int(r[iE] or 0)
        s = float(r[iS] or 0) + float(data[i + 1][iS] or 0)
        a = agg.setdefault(nm, [0, 0.0, 0])
        # a site whose next instruction loops back is a retry loop (executions = retries)
        bm = re.search(r"@!P\d\s+BRA (0x[0-9a-f]+)", data[i + 1][iSrc])
        if bm and int(bm.group(1), 16) < int(r[iA], 16):
            a[2] += e
        a[0] += e
        a[1] += s
    print(f"total samples {tot:.0f}")
    print(f"{'barrier':8s} {'executions':>12s} {'retry-loop execs':>16s} {'samples':>9s} {'% samples':>9s}")
    for nm, (e, s, rl) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{nm:8s} {e:12d} {rl:16d} {s:9.0f} {100 * s / tot:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 6)
