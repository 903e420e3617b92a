# Copy a measurement set (tools/measure_r02.sh output) into profiles/ as
# text: bench lines, the c0 launch list + per-kernel summary, ncu --set full
# summaries (c0 Hessian; c4 Hessian / split TopK / fold), stall tables, the
# GPU test tail, and hessian_traffic.json from the same captures.
#   bash tools/collect_profiles.sh gpurun_out/r02 r02
set -e
I=${1:-gpurun_out/r02}
T=${2:-r02}
P=profiles
for f in $I/bench_*.json; do cp $f $P/${T}_$(basename $f); done
H="# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline (c0, B200; serialised / cold launches: compare shares)"
cp $I/launches_c0.csv $P/${T}_launches_c0.csv
{ echo "$H"; python tools/summarize_launches.py $I/launches_c0.csv; } > $P/${T}_launches_c0.txt
{ echo "# ncu --set full --import-source on --clock-control none -k regex:k_hessian -s 6 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline (c0, B200)";
  ncu -i $I/hessian_c0.ncu-rep --page details; } > $P/${T}_ncu_full_c0.txt
{ echo "# ncu --set full --import-source on --clock-control none -k regex:'k_hessian_ws|k_tks_pass|k_tks_window|k_master_fold' -s 8 -c 4 python tools/profile_round.py c4 (B200)";
  ncu -i $I/c4_kernels.ncu-rep --page details; } > $P/${T}_ncu_full_c4.txt
{ echo "# warp-stall samples of the c0 Hessian capture by SASS window (tools/ncu_stalls.py)";
  python tools/ncu_stalls.py $I/hessian_c0.ncu-rep; } > $P/${T}_hessian_c0_stalls.txt
{ echo "# python -m pytest tests -m gpu -q (B200)"; tail -5 $I/pytest_gpu.log; echo "# smoke()"; cat $I/smoke.log; } > $P/${T}_gputests.txt
python tools/write_traffic.py c0=$I/hessian_c0.ncu-rep c4=$I/c4_kernels.ncu-rep
python - "$T" <<'PY'
import json, sys
t = sys.argv[1]
p = "profiles/hessian_traffic.json"
d = json.load(open(p))
for c in ("c0", "c4"):
    if c in d:
        d[c]["source"] = d[c]["source"].split(" (")[0] + f" (profiles/{t}_ncu_full_{c}.txt, k_hessian_ws section: dram__bytes_read.sum + dram__bytes_write.sum)"
json.dump(d, open(p, "w"), indent=1)
PY
ls -la $P/${T}_*
