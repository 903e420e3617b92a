"""profiles/hessian_traffic.json from ncu --set full captures of k_hessian_ws:
python tools/write_traffic.py c0=path.ncu-rep c4=path.ncu-rep ...
(dram__bytes_read.sum + dram__bytes_write.sum of the one captured launch)."""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(ROOT, "profiles", "hessian_traffic.json")
t = json.load(open(out)) if os.path.exists(out) else {}
t = {k: v for k, v in t.items() if isinstance(v, dict)}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for arg in sys.argv[1:]:
    cfg, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:k_hessian",
                          "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    get = lambda m: float(v[h.index(m)].replace(",", "")) * UNIT[u[h.index(m)]]
    b = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
    t[cfg] = {"bytes_per_launch": int(round(b)),
              "source": f"ncu --set full, one k_hessian_ws launch: dram__bytes_read.sum + dram__bytes_write.sum "
                        f"({os.path.relpath(rep, ROOT)}; kernel duration {v[h.index('gpu__time_duration.sum')]} "
                        f"{u[h.index('gpu__time_duration.sum')]} under the profiler)"}
    print(cfg, t[cfg])
json.dump(t, open(out, "w"), indent=1)
