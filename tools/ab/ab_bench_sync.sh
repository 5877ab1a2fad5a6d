mkdir -p gpurun_out; : > gpurun_out/ab_bs.txt
for cfg in mixtral dsv2 dsv2_lite; do
  python bench.py --config $cfg --no-cpu-baseline --steps 30 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $cfg >> gpurun_out/ab_bs.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print(sys.argv[1], round(d["ms_per_step"], 3), round(d["value"]), d["stages_source"], round(d["stages_ms"]["total"], 3), d["roofline"]["frac"] and round(d["roofline"]["frac"], 3), d["gpu_launches"])
PY
done
