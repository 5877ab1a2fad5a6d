# Layer A/B: send buffer through DRAM (normal) vs an L2-resident window (EPSMOE_DIAG_SEND_WRAP rows; y is
# garbage): the upper bound of keeping the split rows on chip. Interleaved x3, DSv2 bench lines.
set -x
O=gpurun_out/${1:-r02l}
mkdir -p $O
for rep in 1 2 3; do for w in 0 4096; do
  EPSMOE_DIAG_SEND_WRAP=$w timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/wrap=$w /" >> $O/ab.txt
done; done
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum
for w in 0 4096; do
EPSMOE_DIAG_SEND_WRAP=$w timeout 600 ncu --metrics $M --clock-control none -c 12 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_wrap$w.csv 2>/dev/null
done
