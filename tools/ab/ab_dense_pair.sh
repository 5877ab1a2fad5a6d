# Decode batches: router / shared GEMMs on single-CTA 128-row tiles (default below 2048 rows) vs CTA pairs
O=gpurun_out/ab_dense_pair; mkdir -p $O; : > $O/res.txt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_ep.py -q -x 2>&1 | tail -2 >> $O/res.txt
for r in 1 2 3; do for cfg in dsv2_decode mixtral_decode; do for v in 0 2048; do
  EPSMOE_DENSE_PAIR_MIN=$v python bench.py --config $cfg --no-cpu-baseline --steps 50 --e2e-steps 5 > $O/b.json 2>>$O/err.txt
  python - $cfg $v >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_dense_pair/b.json"))
print(sys.argv[1], "pair_min", sys.argv[2], round(d["ms_per_step"], 4), {k: d["stages_ms"][k] for k in ("router", "route", "shared", "gateup", "down", "combine")}, round(d["layer_roofline"]["frac"], 3))
PY
done; done; done
