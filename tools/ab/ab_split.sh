mkdir -p gpurun_out; : > gpurun_out/ab_sp.txt
for r in 1 2; do for sp in 0 1; do
  EPSMOE_SPLIT_REM=$sp python bench.py --config dsv2 --no-cpu-baseline --steps 20 --e2e-steps 2 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $sp >> gpurun_out/ab_sp.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print("split_rem", sys.argv[1], round(d["ms_per_step"], 3), {k: d["stages_ms"][k] for k in ("gateup", "down")}, d["clocks"]["sm_mhz"])
PY
done; done
