# Half tiles in the whole layer: bench lines with EPSMOE_HALF_TILES=0/1, interleaved; GPU suite first
O=gpurun_out/ab_half_layer; mkdir -p $O; : > $O/res.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> $O/res.txt
for r in 1 2 3; do for cfg in dsv2 dsv2_lite mixtral; do for v in 0 1; do
  EPSMOE_HALF_TILES=$v python bench.py --config $cfg --no-cpu-baseline --steps 30 --e2e-steps 2 > $O/b.json 2>>$O/err.txt
  python - $cfg $v >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_half_layer/b.json"))
print(sys.argv[1], "half", sys.argv[2], round(d["ms_per_step"], 3), {k: d["stages_ms"][k] for k in ("shared", "gateup", "down")}, d["clocks"]["sm_mhz"])
PY
done; done; done
