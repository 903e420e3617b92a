"""Where the end-to-end simulate() time goes at a BASELINE config: upload,
state init, the first run (graph capture), steady rounds."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=500)
for rep in range(3):
    t = [time.perf_counter()]
    eng = FedNLEngine(cfg, shards[0].dim, len(shards), max(s.n_samples for s in shards)); t.append(time.perf_counter())
    eng.upload([s.bmat for s in shards], [s.lam for s in shards]); t.append(time.perf_counter())
    eng.init_state(); t.append(time.perf_counter())
    eng.run_rounds(4); t.append(time.perf_counter())
    eng.run_rounds(496); t.append(time.perf_counter())
    eng.close(); t.append(time.perf_counter())
    names = ["create", "upload", "init", "first 4 rounds", "496 rounds", "close"]
    print(rep, " ".join(f"{n}={1e3*(b-a):.1f}ms" for n, a, b in zip(names, t, t[1:])))
