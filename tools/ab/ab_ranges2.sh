# routing ranges target (EPSMOE_RANGES) 2048 vs 8192: ncu durations of gate / scans / permute / combine
O=gpurun_out/ab_ranges2; mkdir -p $O; : > $O/res.txt
for rg in 2048 8192; do for cfg in dsv2 mixtral dsv2_lite; do
  EPSMOE_RANGES=$rg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate_topk|range_scan|seg_scan|permute|combine_kernel" -c 10 --csv \
    --log-file $O/ncu_${cfg}_$rg.csv python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python - $cfg $rg >> $O/res.txt <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(f"gpurun_out/ab_ranges2/ncu_{sys.argv[1]}_{sys.argv[2]}.csv")))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); n = d["Kernel Name"].split("(")[0].split("::")[-1]
        agg.setdefault(n, []).append(float(d["Metric Value"]) / 1e3)
print(sys.argv[1], "ranges", sys.argv[2], {n: round(sorted(v)[len(v) // 2], 1) for n, v in agg.items()})
PY
done; done
