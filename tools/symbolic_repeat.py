"""Warm symbolic phases of config 3 level 1 back to back (device operands),
wall time of each, and with PTAP_TRACE=1 the per-step breakdown on stderr:
python tools/symbolic_repeat.py [alg] [reps]"""
import gc
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen

alg = sys.argv[1] if len(sys.argv) > 1 else "allatonce"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
os.environ.setdefault("PTAP_POOL_KEEP", "1")
ctx = pk.single_rank_context()
a, p = devgen.config_dist("cfg3", 1, 0, ctx.device)
torch.cuda.synchronize()
ts = []
for r in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    plan = pk.run_symbolic(a, p, alg, ctx)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t) * 1e3)
    print(f"run {r}: {ts[-1]:.1f} ms", file=sys.stderr, flush=True)
    del plan
    gc.collect()
print("warm median ms", statistics.median(ts[1:]), "all", [round(x, 1) for x in ts])
