"""Per-panel timeline (globaltimer, us) of the panel-owning solve (fb_solve_phase_cycles)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_08760_b200 import _lib, RunConfig
from paper_2410_08760_b200.engine import FedNLEngine
lib = _lib.load()
buf = (C.c_longlong * (32 + 1024 + 2048))()
for d in [int(a) for a in sys.argv[1:]] or [301]:
    rng = np.random.default_rng(d)
    a = rng.standard_normal((d, d)); spd = a @ a.T / d + np.eye(d)
    iu = np.triu_indices(d); order = np.lexsort((iu[0], iu[1]))
    pk = np.ascontiguousarray(spd[iu[0][order], iu[1][order]]); b = rng.standard_normal(d)
    eng = FedNLEngine(RunConfig(), d, 1, 1)
    cyc = (C.c_longlong * (16 + 64 * 16))(); ms = C.c_float()
    eng.lib.fb_solve_phase_cycles(eng.h, _lib.ptr(pk), 0.0, _lib.ptr(b), 0, cyc, C.byref(ms))
    if os.environ.get("POLLUTE"):  # dirty L2 (as after the Hessian pass) before the timed solve
        import torch
        junk = torch.empty(int(os.environ["POLLUTE"]) << 20, dtype=torch.uint8, device="cuda")
        junk.fill_(1)
        torch.cuda.synchronize()
    eng.lib.fb_solve_phase_cycles(eng.h, _lib.ptr(pk), 0.0, _lib.ptr(b), 0, cyc, C.byref(ms))
    sp = np.array([cyc[16 + i] for i in range(1024)]).reshape(64, 16).astype(np.int64)
    npan = (d + 31) // 32
    t0 = sp[0, 0]
    names = ["fstart", "f_w0done", "A_sync", "w0tile1", "trsm_done", "w0rel", "w0done", "w4done", "bs_own", "bs_recv", "z_done", "st_done", "arr_done", "acc_done", "L2rel", "defer"]
    print(f"d={d} total {ms.value*1e3:.1f} us")
    for p in range(npan):
        print(f"  p={p:2d} " + " ".join((f"{n}={(sp[p, k]-t0)/1e3:7.2f}" if True else "") if sp[p, k] else f"{n}=   -   " for k, n in enumerate(names)))
    print("  rank-0 phase kcycles (mark slots 0..8):", [round(cyc[i] / 1e3, 1) for i in range(9)])
    print("  end-factor %.2f  after-csync %.2f  bs-done %.2f" % tuple((sp[63, k] - t0) / 1e3 for k in range(3)))
    eng.close()
