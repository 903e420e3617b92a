# quick A/B: Hessian-touching parity tests, bench lines, c0 timeline
O=${O:-gpurun_out/q}
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "${TK:-oracle or teacher or simulate_rows or round0_shift or c4 or fold}" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for c in ${CFGS:-c0 c1 c4}; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['kernels_ms'], d['roofline']['frac'])"; done
timeout 120 python tools/timeline.py c0
