mkdir -p gpurun_out; : > gpurun_out/dec.txt
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/dec.txt
for cfg in dsv2_decode mixtral_decode dsv2; do
  python bench.py --config $cfg --no-cpu-baseline --steps 50 --e2e-steps 5 > gpurun_out/dec.json 2>>gpurun_out/dec.err
  python - $cfg >> gpurun_out/dec.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/dec.json"))
print(sys.argv[1], round(d["ms_per_step"], 4), d["stages_ms"], d["layer_roofline"]["bound"], round(d["layer_roofline"]["frac"], 3), round(d["layer_roofline"]["t_roof_ms"], 3), "e2e", round(d["e2e"]["ms_per_step"], 3))
PY
done
