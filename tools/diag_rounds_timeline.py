"""Diagnostic: per-kernel event times in blocks of 10 rounds over a c0 run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=200)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), shards[0].n_samples, lam=shards[0].lam)
eng.upload([s.bmat for s in shards]); eng.init_state()
for blk in range(10):
    b = eng.run_rounds(10, timed=True)
    p = eng.profile()
    f = eng.run_rounds(10)  # the production graph (no per-kernel events)
    print(f"rounds {blk*20:3d}-{blk*20+19:3d} |g|={b.grad_norm[-1]:.2e} " + " ".join(f"{k[3:]}={v*1e3:6.1f}" for k, v in p.items() if k.startswith("ms_"))
          + f" | production round= {1e3 * f.wall_ms[-1] / 10:6.1f}")
