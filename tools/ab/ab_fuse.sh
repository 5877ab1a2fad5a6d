# A/B: ep=1 fused shared-DownGemm + combine (EPSMOE_FUSE_COMBINE) on the bench configs
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "fused or graph or parity" 2>&1 | tail -8 > gpurun_out/ab_pytest.log
for v in 0 1 2 0 1 2; do
  EPSMOE_FUSE_COMBINE=$v python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab_fuse_$v.json 2>>gpurun_out/ab_fuse.err
  python - $v <<'PY' >> gpurun_out/ab_fuse.txt
import json, sys
d = json.load(open(f"gpurun_out/ab_fuse_{sys.argv[1]}.json"))
print("fuse", sys.argv[1], round(d["ms_per_step"], 3), d["stages_ms"], d["clocks"]["sm_mhz"])
PY
done
