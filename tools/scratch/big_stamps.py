import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2410_08760_b200 import CompressorKind, CompressorSpec, RunConfig, _lib
from paper_2410_08760_b200.engine import FedNLEngine
from paper_2410_08760_b200 import data as D
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n, ni = 8, 256
shards = D.gaussian_shards(d, n, ni, 1e-3, seed=3)
cfg = RunConfig(compressor=CompressorSpec(CompressorKind.TOPK, k=8 * d), rounds=30, run_seed=3)
eng = FedNLEngine(cfg, d, n, ni)
eng.upload([s.bmat for s in shards], [s.lam for s in shards])
eng.init_state()
eng.run_rounds(5)
cnt = (C.c_longlong * (32 + 1024 + 2048))()
eng.lib.fb_debug_counters(1, cnt)
eng.run_rounds(3)
eng.lib.fb_debug_counters(0, cnt)
sp = np.array([cnt[32 + 1024 + i] for i in range(8 * ((d + 31) // 32))]).reshape(-1, 8).astype(np.int64)
t0 = sp[0, 0]
for p, r in enumerate(sp):
    prev_end = sp[p - 1, 4] if p else r[0]
    print(p, "gap %.1f load %.1f factor %.1f trsm %.1f update %.1f total %.1f" % (
        (r[0] - prev_end) / 1e3, (r[1] - r[0]) / 1e3, (r[2] - r[1]) / 1e3, (r[3] - r[2]) / 1e3, (r[4] - r[3]) / 1e3, (r[4] - r[0]) / 1e3))
eng.close()
