"""Per-panel timeline (globaltimer, us) of the blocked solve for d > 512
(solve_big.cuh, CTA 0's phase stamps): `python tools/solve_big_timeline.py 1024`
(a small FedNL run at that d: the solve next to a light compressor) or
`... c4` (inside the c4 round, next to the split TopK and the fold)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2410_08760_b200 import CompressorKind, CompressorSpec, RunConfig
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.data import baseline_run_config
from paper_2410_08760_b200.engine import FedNLEngine

arg = sys.argv[1] if len(sys.argv) > 1 else "1024"
if arg == "c4":
    shards = D.baseline_shards("c4")
    cfg = baseline_run_config("c4", rounds=10)
else:
    d = int(arg)
    shards = D.gaussian_shards(d, 8, 256, 1e-3, seed=3)
    cfg = RunConfig(compressor=CompressorSpec(CompressorKind.TOPK, k=8 * d), rounds=30, run_seed=3)
d, n, ni = shards[0].dim, len(shards), shards[0].n_samples
eng = FedNLEngine(cfg, d, n, ni)
eng.upload([s.bmat for s in shards], [s.lam for s in shards])
eng.init_state()
eng.run_rounds(3)
cnt = (C.c_longlong * (32 + 1024 + 2048))()
tl = (C.c_ulonglong * 32)()
eng.lib.fb_debug_timeline(tl)
eng.lib.fb_debug_counters(1, cnt)
eng.run_rounds(1)
eng.lib.fb_debug_counters(0, cnt)
eng.lib.fb_debug_timeline(tl)
npan = (d + 31) // 32
sp = np.array([cnt[32 + 1024 + i] for i in range(8 * npan)]).reshape(-1, 8).astype(np.int64)
t0 = int(tl[2])  # the Hessian pass's first CTA
for i, nm in enumerate(["margins", "hessian", "solve", "solve_wait", "topk", "fold", "finish"]):
    a, b = int(tl[2 * i]), int(tl[2 * i + 1])
    if b and a < (1 << 62):
        print(f"{nm:10s} {(a - t0) / 1e3:10.1f} {(b - t0) / 1e3:10.1f}")
for p, r in enumerate(sp):
    prev_end = sp[p - 1, 4] if p else r[0]
    print(f"panel {p:3d} start {(r[0] - t0) / 1e3:9.1f} gap {(r[0] - prev_end) / 1e3:6.1f} load {(r[1] - r[0]) / 1e3:4.1f} "
          f"factor {(r[2] - r[1]) / 1e3:4.1f} rows {(r[3] - r[2]) / 1e3:4.1f} update {(r[4] - r[3]) / 1e3:4.1f}")
eng.close()
