# router GEMM with the MMA N = E rounded to 16 (this change): GPU suite + ncu router durations
O=gpurun_out/ab_router_n; mkdir -p $O; : > $O/res.txt
for NF in 1 0; do export EPSMOE_ROUTER_NFULL=$NF; echo "[EPSMOE_ROUTER_NFULL=$NF]" >> $O/res.txt
for cfg in dsv2 mixtral dsv2_lite dsv2_decode mixtral_decode; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_kernel -c 12 --csv \
    --log-file $O/ncu_$cfg.csv python bench.py --config $cfg --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 1 --graph off > /dev/null 2>&1
  python - $cfg >> $O/res.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/ab_router_n/ncu_{sys.argv[1]}.csv")))
hdr = None; t = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if "gemm_kernel<2" in d["Kernel Name"] and d["Metric Name"] == "gpu__time_duration.sum": t.append(float(d["Metric Value"]) / 1e3)
print(sys.argv[1], "router us", [round(x, 1) for x in t])
PY
done
done
