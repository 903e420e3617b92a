timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
cp paper_2410_08760_b200/libfednl_b200.so /tmp/cur.so
for v in cur old; do
  if [ $v = cur ]; then cp /tmp/cur.so paper_2410_08760_b200/libfednl_b200.so; else cp tools/probe/lib_$v.so paper_2410_08760_b200/libfednl_b200.so; fi
  echo "== $v"; python tools/timeline.py c0
  for c in c0 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['value'], d['kernels_ms']['hessian'], d['kernels_ms']['round'], d['roofline']['frac'])"; done
done
cp /tmp/cur.so paper_2410_08760_b200/libfednl_b200.so
