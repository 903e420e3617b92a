"""Diagnostic: per-phase cycles of the cluster Cholesky solve for several d / cluster sizes."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_08760_b200 import _lib, RunConfig
from paper_2410_08760_b200.engine import FedNLEngine
names = ["setup", "A", "syncA", "pull", "B", "Bwb", "C", "syncC", "bsolve", "back", "x", "y"] if os.environ.get("CS", "") != "0" else ["setup", "factor_loop", "backsub", "f_warp0", "f_sync", "trsm", "release", "waitL", "apply", "-", "-", "-"]
for d in [int(a) for a in sys.argv[1:]] or [301]:
    rng = np.random.default_rng(d)
    a = rng.standard_normal((d, d)); spd = a @ a.T / d + np.eye(d)
    iu = np.triu_indices(d); order = np.lexsort((iu[0], iu[1]))
    pk = np.ascontiguousarray(spd[iu[0][order], iu[1][order]]); b = rng.standard_normal(d)
    eng = FedNLEngine(RunConfig(), d, 1, 1)
    for cs in [int(x) for x in os.environ.get("CS", "1,2,4,6,8").split(",")]:
        cyc = (C.c_longlong * (16 + 64 * 16))(); ms = C.c_float()
        rc = eng.lib.fb_solve_phase_cycles(eng.h, _lib.ptr(pk), 0.0, _lib.ptr(b), cs, cyc, C.byref(ms))
        print(f"d={d} cluster={cs} rc={rc} {ms.value*1e3:8.1f} us  " + " ".join(f"{n}={c/1e3:.1f}k" for n, c in zip(names, cyc)), flush=True)
