timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in ${@:-c0 c4}; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['kernels_ms'], d['roofline']['frac'])"; done
