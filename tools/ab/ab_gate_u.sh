# gate kernel: 4 tokens at a time (EPSMOE_GATE_U=1, bit-identical) vs one at a time; GPU suite; ncu durations
O=gpurun_out/ab_gate_u; mkdir -p $O; : > $O/res.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> $O/res.txt
for u in 0 1; do for cfg in dsv2 mixtral dsv2_decode; do
  EPSMOE_GATE_U=$u ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate_topk -c 3 --csv \
    --log-file $O/ncu_${cfg}_u$u.csv python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python - $cfg $u >> $O/res.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/ab_gate_u/ncu_{sys.argv[1]}_u{sys.argv[2]}.csv")))
hdr = None; t = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum": t.append(float(d["Metric Value"]))
print(sys.argv[1], "GATE_U", sys.argv[2], "gate_topk us", [round(x / 1e3, 1) for x in t])
PY
done; done
