import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine
shards = D.baseline_shards("c0")
cfg = D.baseline_run_config("c0", rounds=60)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), shards[0].n_samples, lam=shards[0].lam)
eng.upload([s.bmat for s in shards]); eng.init_state()
eng.run_rounds(46)
np.savez_compressed("gpurun_out/diff_r45.npz", d0=eng.round_diff(0), d1=eng.round_diff(1), d2=eng.round_diff(77))
