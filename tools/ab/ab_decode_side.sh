# decode batches: shared experts beside the routed GEMMs (EPSMOE_DECODE_SIDE=1) vs in order; GPU suite first
O=gpurun_out/ab_decode_side; mkdir -p $O; : > $O/res.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> $O/res.txt
for r in 1 2 3; do for cfg in dsv2_decode; do for v in 0 1; do
  EPSMOE_DECODE_SIDE=$v python bench.py --config $cfg --no-cpu-baseline --steps 50 --e2e-steps 5 > $O/b.json 2>>$O/err.txt
  python - $cfg $v >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_decode_side/b.json"))
print(sys.argv[1], "side", sys.argv[2], round(d["ms_per_step"], 4), {k: d["stages_ms"][k] for k in ("router", "route", "shared", "gateup", "down", "combine", "total")}, round(d["layer_roofline"]["frac"], 3))
PY
done; done; done
