# Light DownGemm launches take CTA pairs (this change) - decode and prefill bench lines + GPU suite
O=gpurun_out/ab_down_fill; mkdir -p $O; : > $O/res.txt
python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $O/res.txt
for r in 1 2; do for cfg in mixtral_decode dsv2_decode dsv2_lite; do
  python bench.py --config $cfg --no-cpu-baseline --steps 50 --e2e-steps 5 > $O/b.json 2>>$O/err.txt
  python - $cfg >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_down_fill/b.json"))
print(sys.argv[1], round(d["ms_per_step"], 4), {k: d["stages_ms"][k] for k in ("router", "shared", "gateup", "down")}, round(d["layer_roofline"]["frac"], 3))
PY
done; done
