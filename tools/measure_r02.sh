# Round-2 measurement set (run under gpurun from the repo root): tests, smoke,
# bench lines c0-c4 + the reference arm, the c0 launch list, ncu full-set
# captures of the Hessian (c0, c4) and of the c4 split TopK + fold.
O=${O:-gpurun_out/r02}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for c in c0 c1 c2 c3 c4; do timeout 400 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 400 python bench.py --impl reference > $O/bench_reference_c0.json 2> $O/bench_reference_c0.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_launch.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c0.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/plain_c0.log 2>&1 && \
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_hessian -s 6 -c 1 -o $O/hessian_c0 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full_c0.log 2>&1
python tools/profile_round.py c4 > $O/plain_c4.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_hessian_ws|k_tks_pass|k_tks_window|k_master_fold" -s 8 -c 4 -o $O/c4_kernels python tools/profile_round.py c4 > $O/ncu_full_c4.log 2>&1
echo done > $O/DONE
