# GPU tests + bench line after a change (tag = $1)
set -x
O=gpurun_out/${1:-r02c}
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -25 > $O/pytest_gpu.txt
timeout 600 python bench.py > $O/bench_dsv2.json 2> $O/bench_dsv2.err
