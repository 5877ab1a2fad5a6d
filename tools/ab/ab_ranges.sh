mkdir -p gpurun_out; : > gpurun_out/ab_rg.txt
for r in 1 2; do for rg in 2048 4096 8192; do for ov in 0 1; do
  EPSMOE_RANGES=$rg EPSMOE_OVERLAP_SHARED=$ov python bench.py --config dsv2 --no-cpu-baseline --steps 20 --e2e-steps 2 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $rg $ov >> gpurun_out/ab_rg.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print("ranges", sys.argv[1], "ov", sys.argv[2], round(d["ms_per_step"], 3), {k: d["stages_ms"][k] for k in ("route", "shared", "gateup", "down")}, d["clocks"]["sm_mhz"])
PY
done; done; done
