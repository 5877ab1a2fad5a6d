# E <= 16: CUDA-core router (default) vs the tensor-core router GEMM (EPSMOE_ROUTER_TC=1)
O=gpurun_out/ab_router_small; mkdir -p $O; : > $O/res.txt
python -m pytest tests -m gpu -q -x 2>&1 | tail -4 >> $O/res.txt
for r in 1 2; do for cfg in mixtral_decode mixtral; do for v in 0 1; do
  EPSMOE_ROUTER_TC=$v python bench.py --config $cfg --no-cpu-baseline --steps 30 --e2e-steps 3 > $O/b.json 2>>$O/err.txt
  python - $cfg $v >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_router_small/b.json"))
print(sys.argv[1], "router_tc", sys.argv[2], round(d["ms_per_step"], 4), {k: d["stages_ms"][k] for k in ("router", "route", "gateup", "down", "combine")}, round(d["layer_roofline"]["frac"], 3))
PY
done; done; done
