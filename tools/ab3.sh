cp paper_2410_08760_b200/libfednl_b200.so /tmp/cur.so
for v in cur res5 res8 old; do
  if [ $v = cur ]; then cp /tmp/cur.so paper_2410_08760_b200/libfednl_b200.so; else cp tools/probe/lib_$v.so paper_2410_08760_b200/libfednl_b200.so; fi
  echo "== $v"; python tools/timeline.py c0
  timeout 300 python bench.py --config c0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['kernels_ms']['hessian'], d['kernels_ms']['round'])"
done
cp /tmp/cur.so paper_2410_08760_b200/libfednl_b200.so
