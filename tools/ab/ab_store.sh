# Output-store cost in the expert GEMMs: L2 evict_first hint on the TMA stores vs none vs no stores
# (EPSMOE_GEMM_DIAG=1), with SM clock / power sampled during each run
O=gpurun_out/ab_store; mkdir -p $O; : > $O/gemm.txt
for r in 1 2 3; do
for cfg in dsv2 dsv2_lite; do
for env in "EPSMOE_STORE_HINT=0" "EPSMOE_STORE_HINT=1" "EPSMOE_GEMM_DIAG=1"; do
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 50 > $O/smi.tmp 2>/dev/null &
  SMI=$!
  echo "[$env]" >> $O/gemm.txt
  env $env python tools/gemm_bench.py --config $cfg --reps 30 >> $O/gemm.txt 2>&1
  kill $SMI; wait $SMI 2>/dev/null
  python - >> $O/gemm.txt <<'PY'
import statistics as st
v=[l.split(',') for l in open('gpurun_out/ab_store/smi.tmp') if l.strip()]
c=[float(a) for a,b in v]; p=[float(b) for a,b in v]
hot=[(a,b) for a,b in zip(c,p) if b>400]
if hot: print(f"  clocks: median {st.median(a for a,b in hot):.0f} MHz, power {st.median(b for a,b in hot):.0f} W over {len(hot)} samples")
PY
done; done; done
