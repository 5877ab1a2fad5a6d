# e2e host-slice schedules (EPSMOE_HOST_SLICES; "" = the layer's modelled schedule)
mkdir -p gpurun_out; : > gpurun_out/ab_host.txt
run() {
  EPSMOE_HOST_SLICES="$2" python bench.py --config $1 --no-cpu-baseline --steps 10 --e2e-steps 8 > gpurun_out/ab_host.json 2>>gpurun_out/ab_host.err
  python - "$1" "$2" >> gpurun_out/ab_host.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_host.json"))
print(sys.argv[1], repr(sys.argv[2]), "dev_ms", round(d["ms_per_step"], 2), "e2e_ms", round(d["e2e"]["ms_per_step"], 2), "sm", d["clocks"]["sm_mhz"])
PY
}
for r in 1 2; do
  for s in "" "1,2,3,2" "1,2,4,4,2,1" "1,1,1,1"; do run dsv2 "$s"; done
  for s in "" "1,3,3,1" "1,2,3,2"; do run mixtral "$s"; done
  for s in "" "1,2,2,1" "1,1,1,1"; do run dsv2_lite "$s"; done
done
