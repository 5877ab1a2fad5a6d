mkdir -p gpurun_out; : > gpurun_out/ab_as.txt
python -m pytest tests/test_gpu_parity.py -q -x -k "forward_host" 2>&1 | tail -2 >> gpurun_out/ab_as.txt
for cfg in dsv2 mixtral dsv2_lite; do
  python bench.py --config $cfg --no-cpu-baseline --steps 10 --e2e-steps 8 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $cfg >> gpurun_out/ab_as.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print(sys.argv[1], "dev_ms", round(d["ms_per_step"], 3), "e2e_ms", round(d["e2e"]["ms_per_step"], 3), "e2e tok/s", round(d["e2e"]["value"]))
PY
done
