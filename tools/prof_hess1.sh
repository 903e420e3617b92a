# ncu full-set capture of the Hessian kernel (one launch) at a config
set -e
C=${1:-c0}
python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$C.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_hessian -s 6 -c 1 -o gpurun_out/hess_$C -f python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$C.log 2>&1
