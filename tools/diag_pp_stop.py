import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from test_gpu_parity import sim_case
from conftest import golden
from paper_2410_08760_b200 import simulate
cfg, shards = sim_case("pp_identity_stop")
rows = simulate(cfg, shards)
g = golden("simulate.npz")
for r, gg, ff in zip(rows, g["pp_identity_stop__grad_norm"], g["pp_identity_stop__f_value"]):
    print(r.round, f"{r.grad_norm:.6e} {gg:.6e} dg={abs(r.grad_norm-gg):.2e}  f={r.f_value:.17g} {ff:.17g} df={abs(r.f_value-ff):.2e}")
