"""Stall samples of an ncu --set full capture, by 100-instruction SASS window
and for the hottest instructions: python tools/ncu_stalls.py rep.ncu-rep [kernel-regex]."""
import csv, io, subprocess, sys

rep = sys.argv[1]
kr = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + (["-k", "regex:" + kr] if kr else [])
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
h = rows[1]
end = next((i for i in range(2, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"), len(rows))
data = [r for r in rows[2:end] if len(r) == len(h)]
ix = {k: i for i, k in enumerate(h)}
st = [k for k in h if k.startswith("stall_") and "Not" not in k]
S = lambda r: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tot = sum(S(r) for r in data)
print("samples", tot, "instructions", len(data))
for a in range(0, len(data), 100):
    blk = data[a:a + 100]
    s = sum(S(r) for r in blk)
    if s < 0.01 * tot:
        continue
    agg = {}
    for r in blk:
        for k in st:
            agg[k[6:]] = agg.get(k[6:], 0) + int(r[ix[k]] or 0)
    ops = sorted({(r[ix["Source"]].split()[1] if r[ix["Source"]].split()[0].startswith("@") else r[ix["Source"]].split()[0]).split(".")[0]
                  for r in blk if r[ix["Source"]].split()} & {"DMMA", "STG", "LDG", "STS", "LDS", "DADD", "UTMALDG", "DMUL", "SYNCS", "ATOMG"})
    print(f"{a:5d} {s:6d} {s / tot:.3f}", sorted(agg.items(), key=lambda x: -x[1])[:4], " ".join(ops))
print("hottest:")
for i, r in sorted(enumerate(data), key=lambda x: -S(x[1]))[:25]:
    agg = sorted(((k[6:], int(r[ix[k]] or 0)) for k in st), key=lambda x: -x[1])[:2]
    print(f"{i:5d} {r[ix['Source']].strip()[:60]:60s} {S(r):5d} {r[ix['Instructions Executed']]:>9s} {agg}")
