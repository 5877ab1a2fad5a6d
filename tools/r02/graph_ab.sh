# Host-overhead check: eager forwards vs CUDA-graph replay (same box), DSv2-Lite / DSv2 / Mixtral.
set -x
O=gpurun_out/${1:-r02n}
mkdir -p $O
for rep in 1 2; do for c in dsv2_lite dsv2 mixtral; do for g in off on; do
  timeout 600 python bench.py --config $c --graph $g --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>>$O/err.txt | sed "s/^/$c graph=$g /" >> $O/ab.txt
done; done; done
