"""Stall samples / executed instructions per CUDA source line of an ncu --set full
--import-source on capture: python tools/ncu_lines.py rep.ncu-rep kernel-regex [min-share]."""
import csv, io, subprocess, sys
rep, kr = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kr]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
fname, seen, lines = "", set(), []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Kernel Name" and lines:
        break
    elif len(r) > 8 and r[0].isdigit() and r[2] == "-":
        key = (fname, int(r[0]))
        if key in seen:
            continue
        seen.add(key)
        lines.append((fname, int(r[0]), r[1].strip(), int(r[4] or 0), int(r[7] or 0)))
ts, ti = sum(l[3] for l in lines) or 1, sum(l[4] for l in lines) or 1
print("samples", ts, "warp instructions", ti)
for f, n, src, s, i in sorted(lines, key=lambda l: (l[0], l[1])):
    if s >= thr * ts or i >= thr * ti:
        print(f"{f}:{n:5d} {s / ts:6.3f} {i / ti:6.3f}  {src[:90]}")
if len(sys.argv) > 4:  # range sums: file:lo-hi,...
    for spec in sys.argv[4].split(","):
        f, rg = spec.split(":")
        lo, hi = map(int, rg.split("-"))
        s = sum(l[3] for l in lines if l[0].startswith(f) and lo <= l[1] <= hi)
        i = sum(l[4] for l in lines if l[0].startswith(f) and lo <= l[1] <= hi)
        print(f"{spec:40s} samples {s / ts:6.3f} instr {i / ti:6.3f}")
