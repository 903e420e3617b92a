"""A few production rounds of a BASELINE config (the target of the ncu captures
in tools/measure_r02.sh), then the event-instrumented per-kernel times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=10)
eng = FedNLEngine(cfg, shards[0].dim, len(shards), max(s.n_samples for s in shards),
                  topk_path=int(os.environ.get("TOPK_PATH", "0")))
eng.upload([s.bmat for s in shards], [s.lam for s in shards])
eng.init_state()
eng.run_rounds(int(os.environ.get("WARM", "2")))
eng.run_rounds(int(os.environ.get("ROUNDS", "2")), timed=True)
print(name, "event profile (ms):", {k: round(v, 4) for k, v in eng.profile().items() if k.startswith("ms_")})
eng.close()
