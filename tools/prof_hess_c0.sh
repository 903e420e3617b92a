# ncu full-set capture of one Hessian launch of a config (after a clean run)
O=${O:-gpurun_out/ph}
C=${CFG:-c0}
mkdir -p $O
python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > $O/plain_$C.log 2>&1 && \
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_hessian -s ${SKIP:-6} -c 1 -o $O/hessian_$C python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_$C.log 2>&1
tail -3 $O/ncu_$C.log
