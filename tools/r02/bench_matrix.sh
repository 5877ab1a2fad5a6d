# Smoke of bench.py's options on one GPU: every line must parse and carry the contract keys.
O=gpurun_out/${1:-r02bm}
mkdir -p $O
: > $O/summary.txt
run() {
  echo "== $*" >> $O/err.txt
  timeout 300 python bench.py "$@" --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/line.json 2>> $O/err.txt
  rc=$?
  python -c "
import json,sys
try:
    d=json.loads(open('$O/line.json').read().strip().splitlines()[-1])
    ok=all(k in d for k in ('metric','value','unit','roofline','e2e','gpu_launches'))
    print('rc=$rc', 'ok' if ok else 'MISSING', round(d['value']), d['ms_per_step'] and round(d['ms_per_step'],3), '$*')
except Exception as e:
    print('rc=$rc', 'FAIL', repr(e)[:80], '$*')
" >> $O/summary.txt
}
run --config tiny
run --config dsv2_lite
run --config dsv2_lite --skew 1.0
run --config dsv2_lite --chunks 4
run --config dsv2_lite --kind dense
run --config dsv2_lite --kind grouped --chunks 8
run --config dsv2_lite --dispatch-fp8
run --config dsv2_lite --local-reduce
run --config dsv2_lite --route-groups 8 --route-topk-groups 3
run --config dsv2_lite --sm-gemm 132
run --config dsv2_lite --tile-m 128
run --config mixtral --chunks 2 --token-slices 2
run --config dsv2_decode --graph off
run --config mixtral_decode --graph on
run --config dsv2 --skew 0.5 --chunks 5
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > $O/ref.json 2>> $O/err.txt; echo "reference rc=$? $(head -c 200 $O/ref.json)" >> $O/summary.txt
