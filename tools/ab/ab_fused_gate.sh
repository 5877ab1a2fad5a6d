# topKGating fused into the router GEMM epilogue (EPSMOE_FUSED_GATE=1) vs the separate gate kernel
O=gpurun_out/ab_fused_gate; mkdir -p $O; : > $O/res.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 >> $O/res.txt
for r in 1 2; do for cfg in mixtral dsv2 mixtral_decode dsv2_decode; do for v in 0 1; do
  EPSMOE_FUSED_GATE=$v python bench.py --config $cfg --no-cpu-baseline --steps 30 --e2e-steps 2 > $O/b.json 2>>$O/err.txt
  python - $cfg $v >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_fused_gate/b.json"))
print(sys.argv[1], "fused", sys.argv[2], round(d["ms_per_step"], 4), {k: d["stages_ms"][k] for k in ("router", "route", "shared", "gateup")})
PY
done; done; done
