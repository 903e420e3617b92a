"""Per-CTA [start, end] of the instrumented compressor kernel in the LAST of
R back-to-back production rounds: python tools/spans.py c0 [R] [topk_path]."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_08760_b200 import _lib, data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
tp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=R + 10)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), max(s.n_samples for s in shards), topk_path=tp)
eng.upload([s.bmat for s in shards], [s.lam for s in shards]); eng.init_state()
eng.run_rounds(5)
lib = _lib.load()
cnt = (C.c_longlong * (32 + 1024 + 2048))()
tl = (C.c_ulonglong * 32)()
for mode in ("single", "back-to-back"):
    lib.fb_debug_timeline(tl)
    lib.fb_debug_counters(1, cnt)
    if mode == "single":
        for _ in range(3):
            eng.run_rounds(1)
    else:
        eng.run_rounds(R)
    lib.fb_debug_counters(0, cnt)
    lib.fb_debug_timeline(tl)
    if mode != "single":
        first = tl[0]
        lastm = cnt[32 + 1024 + 2048 - 32]
        print(f"round period (margins start to margins start): {(lastm - first) / 1e3 / (R - 1):.1f} us")
    sp = np.array([cnt[32 + 1024 + i] for i in range(2 * len(shards))]).reshape(-1, 2).astype(np.int64)
    t0 = sp[:, 0].min()
    st, en = (sp[:, 0] - t0) / 1e3, (sp[:, 1] - t0) / 1e3
    dur = en - st
    print(f"{mode}: start min/med/max {st.min():.1f}/{np.median(st):.1f}/{st.max():.1f} us; end max {en.max():.1f}; "
          f"duration min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us")
names = ["margins", "hessian", "solve", "solve_wait", "topk", "fold", "finish", "reduce_done", "factor_done", "red_loads", "red_clients", "red_csync", "k_reduce", "ls_trials", "ls_decide", "-"]
last = np.array([cnt[32 + 1024 + 2048 - 32 + i] for i in range(32)]).reshape(16, 2).astype(np.int64)
t0 = last[0, 0]
print("last round (latest start / end, us from margins' latest start):")
for i, nm in enumerate(names):
    if last[i, 1]:
        print(f"  {nm:12s} {(last[i,0]-t0)/1e3 if last[i,0] else float('nan'):8.1f} {(last[i,1]-t0)/1e3:8.1f}")
