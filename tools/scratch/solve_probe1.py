import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_08760_b200 import CompressorKind, CompressorSpec, RunConfig
from paper_2410_08760_b200.engine import FedNLEngine
from paper_2410_08760_b200 import data as D
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n, ni = 8, 256
shards = D.gaussian_shards(d, n, ni, 1e-3, seed=3)
cfg = RunConfig(compressor=CompressorSpec(CompressorKind.TOPK, k=8 * d), rounds=30, run_seed=3)
eng = FedNLEngine(cfg, d, n, ni)
eng.upload([s.bmat for s in shards], [s.lam for s in shards])
eng.init_state()
eng.run_rounds(3)
eng.close()
