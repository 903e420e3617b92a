"""Diagnostic: wall-clock phases of one simulate()-equivalent call at c0."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_08760_b200 import data as D, simulate
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=100)
d, n, ni = shards[0].dim, len(shards), shards[0].n_samples
simulate(cfg, shards)  # warm process-wide state (context, module load)
for rep in range(2):
    t = [time.perf_counter()]
    eng = FedNLEngine(cfg, d, n, ni, lam=shards[0].lam); t.append(time.perf_counter())
    eng.upload([s.bmat for s in shards]); t.append(time.perf_counter())
    eng.init_state(); t.append(time.perf_counter())
    b = eng.run_rounds(100); t.append(time.perf_counter())
    eng.final_eval(); t.append(time.perf_counter())
    eng.close(); t.append(time.perf_counter())
    names = ["create", "upload", "init", "rounds", "final", "close"]
    print(" ".join(f"{k}={1e3*(t[i+1]-t[i]):.2f}ms" for i, k in enumerate(names)), f"device={b.wall_ms[-1]:.2f}ms")
t0 = time.perf_counter(); simulate(cfg, shards); print("simulate ms", 1e3 * (time.perf_counter() - t0))
