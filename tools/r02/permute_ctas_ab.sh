# The split (permute) on a capped persistent grid while the shared GEMMs run: per-SM contention vs energy.
set -x
O=gpurun_out/${1:-r02z}
mkdir -p $O
for rep in 1 2 3; do for v in 0 16 32 64; do
  EPSMOE_PERMUTE_CTAS=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/ctas=$v /" >> $O/ab.txt
done; done
