"""Diagnostic: replay the golden compressor cases one call at a time, printing each."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2410_08760_b200 import leaf, CompressorSpec, CompressorKind
g = np.load(os.path.join(ROOT, "tests/golden/compress.npz"))
for name in g["case_names"].tolist():
    pk = g[f"{name}__input"]; d = int(g[f"{name}__d"])
    for key in g.files:
        if not (key.startswith(name + "__") and key.endswith("__val")):
            continue
        tag = key[len(name) + 2:-5]
        parts = tag.split("__"); kind = parts[0]; weighted = kind.endswith("W"); kind = kind.rstrip("W")
        if kind in ("identity", "natural"):
            k, seed = None, int(parts[1][1:])
        else:
            k, seed = int(parts[1][1:]), int(parts[2][1:])
        print(name, tag, flush=True)
        delta = leaf.compress_packed_batch(pk[None, :], d, CompressorSpec(CompressorKind(kind), k=k, topk_weighted=weighted), [seed])[0]
        ok = np.array_equal(delta.values, g[f"{name}__{tag}__val"])
        if not ok:
            print("   MISMATCH", delta.values[:8], g[f"{name}__{tag}__val"][:8], flush=True)
