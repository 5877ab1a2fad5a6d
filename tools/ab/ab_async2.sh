mkdir -p gpurun_out; : > gpurun_out/ab_as2.txt
for cfg in dsv2 mixtral; do for sch in "" "1" "1,8,1" "1,4,1" "1,2,8,2,1" "1,2,4,4,2,1"; do
  EPSMOE_HOST_SLICES="$sch" python bench.py --config $cfg --no-cpu-baseline --steps 5 --e2e-steps 8 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $cfg "$sch" >> gpurun_out/ab_as2.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print(sys.argv[1], repr(sys.argv[2]), "dev_ms", round(d["ms_per_step"], 3), "e2e_ms", round(d["e2e"]["ms_per_step"], 3))
PY
done; done
