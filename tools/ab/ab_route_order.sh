# Shared experts concurrent with routing (default) vs in order with more routing ranges
O=gpurun_out/ab_route_order; mkdir -p $O; : > $O/res.txt
for r in 1 2 3 4; do
for env in "EPSMOE_OVERLAP_SHARED=1" "EPSMOE_OVERLAP_SHARED=0 EPSMOE_RANGES=8192" "EPSMOE_OVERLAP_SHARED=0 EPSMOE_RANGES=16384" "EPSMOE_OVERLAP_SHARED=1 EPSMOE_RANGES=8192"; do
  env $env python bench.py --config dsv2 --no-cpu-baseline --steps 20 --e2e-steps 2 > $O/b.json 2>>$O/err.txt
  python - "$env" >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_route_order/b.json"))
print(f"[{sys.argv[1]}]", round(d["ms_per_step"], 3), {k: d["stages_ms"][k] for k in ("route", "shared", "gateup", "down")}, d["clocks"]["sm_mhz"])
PY
done; done
