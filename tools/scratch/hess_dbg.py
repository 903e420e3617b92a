import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.data import baseline_run_config
from paper_2410_08760_b200.engine import FedNLEngine
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c0"
shards = D.baseline_shards(cfgname)
cfg = baseline_run_config(cfgname, rounds=40)
d, n, ni = shards[0].dim, len(shards), shards[0].n_samples
eng = FedNLEngine(cfg, d, n, ni)
eng.upload([s.bmat for s in shards], [s.lam for s in shards])
eng.init_state()
eng.run_rounds(4)
cnt = (C.c_longlong * (32 + 1024 + 2048))()
eng.lib.fb_debug_counters(1, cnt)
R = 8
eng.run_rounds(R)
eng.lib.fb_debug_counters(0, cnt)
epi, ntile, wt, nw, ml = cnt[11], cnt[12], cnt[13], cnt[14], cnt[15]
print(f"tiles/round {ntile / R:.0f}; epilogue cycles/tile {epi / max(ntile,1):.0f}; DMMA warp0: items/round {nw / R:.0f}, "
      f"cs_empty wait cycles/item {wt / max(nw,1):.0f}, mainloop cycles/item {ml / max(nw,1):.0f}")
print(f"first-stage wait cycles/item {cnt[18] / max(nw,1):.0f}; hand-off (wait + stores + arrive) cycles/item {cnt[19] / max(nw,1):.0f}")
eng.close()
