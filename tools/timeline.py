"""Per-kernel [first start, last end] of single production-graph rounds
(globaltimer, fb_debug_timeline), relative to the round's margins start."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_08760_b200 import _lib, data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=10)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), max(s.n_samples for s in shards))
eng.upload([s.bmat for s in shards], [s.lam for s in shards]); eng.init_state()
eng.run_rounds(5)
lib = _lib.load()
buf = (C.c_ulonglong * 32)()
cnt = (C.c_longlong * (32 + 1024 + 2048))()
names = ["margins", "hessian", "solve", "solve_wait", "topk", "fold", "finish", "reduce_done", "factor_done", "red_loads", "red_clients", "red_csync", "k_reduce", "ls_trials", "ls_decide"]
acc = {}
for rep in range(8):
    lib.fb_debug_timeline(buf)           # re-arm
    lib.fb_debug_counters(1, cnt)        # g_dbg_on = 1
    eng.run_rounds(1)
    lib.fb_debug_counters(0, cnt)
    lib.fb_debug_timeline(buf)
    t0 = min(buf[2 * s] for s in range(16) if buf[2 * s] != 2**64 - 1)
    for s, nm in enumerate(names):
        a, b = buf[2 * s], buf[2 * s + 1]
        if b == 0:
            continue
        acc.setdefault(nm, []).append((((a - t0) / 1e3) if a != 2**64 - 1 else float("nan"), (b - t0) / 1e3))
for nm in names:
    if nm in acc:
        v = np.array(acc[nm])
        print("%-11s start %7.1f  end %7.1f  (us, median of %d rounds)" % (nm, np.median(v[:, 0]), np.median(v[:, 1]), len(v)))
