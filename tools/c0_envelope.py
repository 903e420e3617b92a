"""Print the GPU's c0 trajectory next to the reference's 1- and 8-thread ones."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from cases_r2 import case_r2, run_config
from paper_2410_08760_b200 import simulate
g = np.load("tests/golden/simulate_r2.npz")
kw, shards = case_r2("c0_r20")
rows = simulate(run_config(kw), shards)
g1, g8 = g["c0_r20__grad_norm"], g["c0_r20_mt__grad_norm"]
for i, r in enumerate(rows):
    print(i, r.grad_norm, "rel1 %.2e rel8 %.2e env %.2e" % (abs(r.grad_norm - g1[i]) / g1[i], abs(r.grad_norm - g8[i]) / g8[i], abs(g1[i] - g8[i]) / g1[i]))
f1, f8 = g["c0_r20__f_value"], g["c0_r20_mt__f_value"]
for i, r in enumerate(rows):
    print(i, "f rel1 %.2e rel8 %.2e env %.2e" % (abs(r.f_value - f1[i]) / f1[i], abs(r.f_value - f8[i]) / f8[i], abs(f1[i] - f8[i]) / f1[i]))
