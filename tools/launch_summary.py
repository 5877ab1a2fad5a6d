#!/usr/bin/env python
"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`): the
last full-size layer forward (forwards start at a router GEMM launch; the host
API's token-sliced calls make shorter ones, so the last forward of the largest
serialised time is taken), per kernel, in us, with its share of the serialised
sum.

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
    segs = [recs[a:b] for a, b in zip(starts, starts[1:] + [len(recs)])] or [recs]
    # drop trailing non-layer launches (e.g. generator fills) from each segment's end
    tot = [sum(v for n, v in sg if "epsmoe" in n) for sg in segs]
    big = max(tot)
    last = [sg for sg, t in zip(segs, tot) if t >= 0.9 * big][-1]
    last = [(n, v) for n, v in last if "epsmoe" in n]
    # a forward ends at its combine: small host-call slices launch their shared experts before
    # their router, so anything after the combine belongs to the next forward
    ends = [i for i, (n, _) in enumerate(last) if "combine" in n]
    if ends:
        last = last[:ends[-1] + 1]
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
