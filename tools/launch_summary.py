#!/usr/bin/env python
"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`): the
last layer forward (from the last router GEMM launch on), per kernel, in us,
with its share of the serialised sum.

  python tools/launch_summary.py profiles/r02k_launches_dsv2.csv
"""
import csv
import sys
from collections import OrderedDict


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    iname, ival = h.index("Kernel Name"), h.index("Metric Value")
    recs = [(r[iname], float(r[ival].replace(",", ""))) for r in rows[1:] if len(r) > ival]
    starts = [i for i, (n, _) in enumerate(recs) if "gemm_kernel<2" in n]
    last = recs[starts[-1]:] if starts else recs
    agg = OrderedDict()
    for n, v in last:
        key = n.split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("unnamed>::", "")
        if key.startswith("gemm_kernel"):
            key = n.split(">(")[0].replace("void ", "").replace("<unnamed>::", "").replace("unnamed>::", "") + ">"
        t, c = agg.get(key, (0.0, 0))
        agg[key] = (t + v, c + 1)
    tot = sum(t for t, _ in agg.values())
    for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{t / 1e3:10.1f} us  {100 * t / tot:5.1f}%  x{c:<3d} {k}")
    print(f"{tot / 1e3:10.1f} us  total ({len(last)} launches)")


if __name__ == "__main__":
    main(sys.argv[1])
