mkdir -p gpurun_out; : > gpurun_out/ab_gather.txt
for cfg in dsv2_lite mixtral dsv2; do for g in 0 1; do
  EPSMOE_GATHER=$g python bench.py --config $cfg --no-cpu-baseline --steps 10 --e2e-steps 2 > gpurun_out/ab_gather.json 2>>gpurun_out/ab_gather.err
  python - $g $cfg >> gpurun_out/ab_gather.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_gather.json"))
print(sys.argv[2], "gather", sys.argv[1], round(d["ms_per_step"], 3), d["stages_ms"])
PY
done; done
