mkdir -p gpurun_out; : > gpurun_out/ab_ov.txt
for r in 1 2 3; do for ov in 0 1; do
  EPSMOE_OVERLAP_SHARED=$ov python bench.py --config dsv2 --no-cpu-baseline --steps 20 --e2e-steps 2 > gpurun_out/ab_ov.json 2>>gpurun_out/ab_ov.err
  python - $ov >> gpurun_out/ab_ov.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_ov.json"))
print("overlap", sys.argv[1], round(d["ms_per_step"], 3), d["stages_ms"], d["clocks"]["sm_mhz"])
PY
done; done
