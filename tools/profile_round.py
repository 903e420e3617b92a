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
eng.run_rounds(int(os.environ.get("WARM", "3")))
lib = _lib.load()
buf = (C.c_longlong * (32 + 1024 + 2048))()
lib.fb_debug_counters(1, buf)
R = 5
eng.run_rounds(R, timed=True)
print("event profile (ms):", {k: round(v, 4) for k, v in eng.profile().items() if k.startswith("ms_")})
lib.fb_debug_counters(0, buf)
print("hessian CTA-avg cycles: mainloop %.0f epilogue %.0f (CTAs %.0f)" % (buf[20] / max(buf[22], 1), buf[21] / max(buf[22], 1), buf[22] / R))
print(name, "per-round cycles (k):", [round(buf[i] / R / 1e3, 1) for i in range(16)], "not-take-all CTAs:", buf[16] / R)
print("slots 24-28 (k):", [round(buf[i] / R / 1e3, 1) for i in range(24, 29)])
cta = np.array([buf[32 + i] for i in range(len(shards))]) / 1e3
print("last round per-CTA kcycles: min %.1f median %.1f max %.1f" % (cta.min(), np.median(cta), cta.max()))
print("slowest clients", np.argsort(-cta)[:8], np.sort(cta)[::-1][:8])
span = np.array([buf[32 + 1024 + i] for i in range(2 * len(shards))]).reshape(-1, 2)
st, en = span[:, 0], span[:, 1]
print("last round TopK span us: %.1f (starts spread %.1f us, per-CTA %.1f..%.1f us)" % ((en.max() - st.min()) / 1e3, (st.max() - st.min()) / 1e3, ((en - st).min()) / 1e3, ((en - st).max()) / 1e3))
