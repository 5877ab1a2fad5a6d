mkdir -p gpurun_out; : > gpurun_out/ab_g.txt
for cfg in dsv2_decode mixtral_decode; do for g in off on; do
  python bench.py --config $cfg --no-cpu-baseline --graph $g --steps 50 --e2e-steps 5 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $cfg $g >> gpurun_out/ab_g.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print(sys.argv[1], "graph", sys.argv[2], round(d["ms_per_step"], 4), d["gpu_launches"], d["config"]["cuda_graph"], round(d["stages_ms"]["total"], 4))
PY
done; done
