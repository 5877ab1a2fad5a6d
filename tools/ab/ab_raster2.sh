mkdir -p gpurun_out; : > gpurun_out/ab_r2.txt
for r in 1 2; do for cfg in dsv2 mixtral dsv2_lite; do for gm in 0 4; do
  EPSMOE_RASTER_GM=$gm python bench.py --config $cfg --no-cpu-baseline --steps 20 --e2e-steps 2 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $cfg $gm >> gpurun_out/ab_r2.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print(sys.argv[1], "gm", sys.argv[2], round(d["ms_per_step"], 3), {k: d["stages_ms"][k] for k in ("gateup", "down", "shared", "route")}, d["clocks"]["sm_mhz"])
PY
done; done; done
