"""PhaseClock cycles (g_dbg slots, CTA 0 of the instrumented kernels) per round
of a BASELINE config's production graph: python tools/phases.py c0 [rounds]."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_08760_b200 import _lib, data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=R + 10)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), max(s.n_samples for s in shards),
                  topk_path=int(os.environ.get("TOPK_PATH", "0")))
eng.upload([s.bmat for s in shards], [s.lam for s in shards]); eng.init_state()
eng.run_rounds(5)
lib = _lib.load()
cnt = (C.c_longlong * (32 + 1024 + 2048))()
lib.fb_debug_counters(1, cnt)
eng.run_rounds(R)
lib.fb_debug_counters(0, cnt)
print(name, "kcycles per round, slot: value", {i: round(cnt[i] / R / 1e3, 2) for i in range(32) if cnt[i]})
