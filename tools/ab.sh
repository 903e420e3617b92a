set -x
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t2.log 2>&1; tail -3 gpurun_out/t2.log
for c in c0 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c NEW', d['value'], d['kernels_ms'], d['roofline']['frac'])"; done
cp paper_2410_08760_b200/libfednl_b200.so /tmp/new.so; cp tools/probe/lib_old.so paper_2410_08760_b200/libfednl_b200.so
for c in c0 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c OLD', d['value'], d['kernels_ms'], d['roofline']['frac'])"; done
cp /tmp/new.so paper_2410_08760_b200/libfednl_b200.so
