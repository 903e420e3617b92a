import os, sys, subprocess
sys.path.insert(0, "/root/repo")
code = r'''
import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2410_08760_b200 import data as D, simulate
from paper_2410_08760_b200.engine import FedNLEngine
shards = D.baseline_shards("c0")
cfg = D.baseline_run_config("c0", rounds=3)
rows = simulate(cfg, shards)
print([r.bytes_up_cum for r in rows])
eng = FedNLEngine(cfg, shards[0].dim, len(shards), shards[0].n_samples, lam=shards[0].lam)
eng.upload([s.bmat for s in shards]); eng.init_state()
b = eng.run_rounds(1)
cnt = b.entry_counts[0] if hasattr(b, "entry_counts") else None
print("counts", None if cnt is None else (int(cnt.min()), int(cnt.max()), int((cnt != 2408).sum())))
'''
for env in ({"FB_TOPK_SPLIT": "0"}, {"FB_TOPK_SPLIT": "1"}, {"FB_TOPK_SPLIT": "1", "FB_SERIAL_ROUND": "1"}):
    e = dict(os.environ); e.update(env)
    out = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True)
    print(env, out.stdout.strip(), out.stderr.strip()[-300:])
