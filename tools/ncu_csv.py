"""Summarise an `ncu --csv --metrics ...` capture: one line per launch."""
import csv
import io
import sys

for path in sys.argv[1:]:
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
    hdr, agg = rows[0], {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        agg.setdefault((int(d["ID"]), d["Kernel Name"].split("(")[0]), {})[d["Metric Name"]] = d["Metric Value"]
    for (i, k), m in sorted(agg.items()):
        print(path.split("/")[-1], i, k, " ".join(f"{a.split('.')[0]}={b}" for a, b in m.items()))
