"""Diagnostic: run every compressor kind once on small inputs (one process per kind)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_08760_b200 import leaf, CompressorSpec, CompressorKind
kind = sys.argv[1]
d = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = d * (d + 1) // 2
rng = np.random.default_rng(0)
P = rng.standard_normal((1, w))
k = None if kind in ("identity", "natural") else max(1, w // 3)
out = leaf.compress_packed_batch(P, d, CompressorSpec(CompressorKind(kind), k=k), [77])
print(kind, d, "ok", out[0].entry_count, out[0].draws)
