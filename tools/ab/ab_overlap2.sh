# shared experts concurrent with routing (default) vs in order, current kernels; interleaved rounds
O=gpurun_out/ab_overlap2; mkdir -p $O; : > $O/res.txt
for r in 1 2 3 4 5; do for ov in 0 1; do for cfg in dsv2 dsv2_lite; do
  EPSMOE_OVERLAP_SHARED=$ov python bench.py --config $cfg --no-cpu-baseline --steps 30 --e2e-steps 2 > $O/b.json 2>>$O/err.txt
  python - $cfg $ov >> $O/res.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_overlap2/b.json"))
print(sys.argv[1], "overlap", sys.argv[2], round(d["ms_per_step"], 3), {k: d["stages_ms"][k] for k in ("router", "route", "shared", "gateup", "down")}, d["clocks"]["sm_mhz"])
PY
done; done; done
