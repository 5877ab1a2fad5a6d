mkdir -p gpurun_out; : > gpurun_out/ab_cs.txt
python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> gpurun_out/ab_cs.txt
for r in 1 2; do for n in 1 4 8; do for cs in 1 2; do
  EPSMOE_CHUNK_STREAMS=$cs python bench.py --config dsv2 --chunks $n --kind grouped --no-cpu-baseline --steps 15 --e2e-steps 2 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $n $cs >> gpurun_out/ab_cs.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print("chunks", sys.argv[1], "streams", sys.argv[2], round(d["ms_per_step"], 3), d["clocks"]["sm_mhz"])
PY
done; done; done
