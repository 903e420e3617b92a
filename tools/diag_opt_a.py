import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2410_08760_b200 import leaf
m = leaf.eigen_clamp_min(np.diag([-1.0, 4.0]), 0.5)
print("clamp", m.tolist())
print("jacobi", [x.tolist() for x in leaf.jacobi_eigh(np.diag([-1.0, 4.0]))])
try:
    print("solve", leaf.cholesky_solve(m, np.array([1.0, 8.0])).tolist())
except Exception as e:
    print("ERR", e)
print("solve diag", leaf.cholesky_solve(np.diag([0.5, 4.0]), np.array([1.0, 8.0])).tolist())
