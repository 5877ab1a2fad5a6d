# Layer A/B, 5 interleaved rounds: DownGemm static (EPSMOE_DYN_SCHED=2) vs all dynamic (1).
O=gpurun_out/${1:-r02x}
mkdir -p $O
for rep in 1 2 3 4 5; do for v in 1 2; do for c in dsv2 dsv2_lite; do
  EPSMOE_DYN_SCHED=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/dyn=$v /" >> $O/ab.txt
done; done; done
