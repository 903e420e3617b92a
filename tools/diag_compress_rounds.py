"""Diagnostic: per-chunk compressor / fold times over many rounds, with the
split TopK's fallback counter (g_dbg[17])."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_08760_b200 import _lib, data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 300
CH = int(sys.argv[3]) if len(sys.argv) > 3 else 50
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=R)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), shards[0].n_samples, lam=shards[0].lam)
eng.upload([s.bmat for s in shards]); eng.init_state()
lib = _lib.load()
buf = (C.c_longlong * (32 + 1024 + 2048))()
for r0 in range(0, R, CH):
    lib.fb_debug_counters(1, buf)
    b = eng.run_rounds(CH, timed=True)
    lib.fb_debug_counters(0, buf)
    p = eng.profile()
    print(r0, "grad %.3e" % b.grad_norm[-1], {k: round(v, 4) for k, v in p.items() if k in ("ms_compress", "ms_fold", "ms_solve", "ms_round")},
          "fallback CTAs", buf[17], "over/G>=k/short/list", [buf[i] for i in range(24, 28)], flush=True)
