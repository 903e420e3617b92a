"""Diagnostic: phase clocks of instrumented kernels over a few c0 rounds."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_08760_b200 import _lib, data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=10)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), shards[0].n_samples, lam=shards[0].lam)
eng.upload([s.bmat for s in shards]); eng.init_state()
eng.run_rounds(3)
lib = _lib.load()
buf = (C.c_longlong * 32)()
lib.fb_debug_counters(1, buf)
R = 5
eng.run_rounds(R)
lib.fb_debug_counters(0, buf)
print(name, "per-round cycles (k):", [round(buf[i] / R / 1e3, 1) for i in range(16)])
