# Decode batches: routed-expert tile rows by R14 (auto = 128 below 512 rows/expert) vs forced 256 (CTA pairs)
O=gpurun_out/ab_decode_tile; mkdir -p $O; : > $O/res.txt
for r in 1 2 3; do for cfg in dsv2_decode mixtral_decode; do for tm in 0 256; do
  python bench.py --config $cfg --no-cpu-baseline --steps 50 --e2e-steps 5 --tile-m $tm > $O/b.json 2>>$O/err.txt
  python - $cfg $tm >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_decode_tile/b.json"))
print(sys.argv[1], "tile_m", sys.argv[2], round(d["ms_per_step"], 4), {k: d["stages_ms"][k] for k in ("router", "shared", "gateup", "down")}, round(d["layer_roofline"]["frac"], 3))
PY
done; done; done
