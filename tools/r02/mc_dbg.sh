set -x
O=gpurun_out/${1:-r02t}
mkdir -p $O
EPSMOE_DEBUG_LAUNCH=1 EPSMOE_MC=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "grouped_gemm" 2>&1 | tail -30 > $O/pytest_mc.txt
EPSMOE_DEBUG_LAUNCH=1 EPSMOE_MC=0 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "grouped_gemm" 2>&1 | tail -30 > $O/pytest_mc0.txt
