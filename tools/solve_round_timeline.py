"""Per-panel timeline (us) of the panel-owning solve INSIDE the production
round (stamps written while g_dbg_on), last round of R: python tools/solve_round_timeline.py c0."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_08760_b200 import _lib, data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=40)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), max(s.n_samples for s in shards))
eng.upload([s.bmat for s in shards], [s.lam for s in shards]); eng.init_state()
eng.run_rounds(5)
lib = _lib.load()
cnt = (C.c_longlong * (32 + 1024 + 2048))()
lib.fb_debug_counters(1, cnt)
eng.run_rounds(1)
lib.fb_debug_counters(0, cnt)
sp = np.array([cnt[32 + i] for i in range(1024)]).reshape(64, 16).astype(np.int64)
npan = (shards[0].dim + 31) // 32
t0 = sp[0, 0]
names = ["fstart", "f_w0done", "A_sync", "w0tile1", "trsm_done", "w0rel", "w0done", "w4done", "bs_own", "bs_recv", "z_done", "st_done", "arr_done", "acc_done", "L2rel", "defer"]
for p in range(npan):
    print(f"  p={p:2d} " + " ".join(f"{n}={(sp[p, k]-t0)/1e3:6.2f}" if sp[p, k] else f"{n}=  -   " for k, n in enumerate(names)))
