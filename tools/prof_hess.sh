# ncu full-set captures of the Hessian kernel at c0 (new build, then the old build)
set -e
python bench.py --config c0 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_new.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_hessian -s 6 -c 1 -o gpurun_out/hess_new_c0 -f python bench.py --config c0 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_new.log 2>&1
cp paper_2410_08760_b200/libfednl_b200.so /tmp/new.so; cp tools/probe/lib_old.so paper_2410_08760_b200/libfednl_b200.so
python bench.py --config c0 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_old.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_hessian -s 6 -c 1 -o gpurun_out/hess_old_c0 -f python bench.py --config c0 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_old.log 2>&1
cp /tmp/new.so paper_2410_08760_b200/libfednl_b200.so
