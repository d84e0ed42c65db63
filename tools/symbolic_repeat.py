"""Repeated symbolic phases of one algorithm (PTAP_TRACE=1 for the phase and
pool breakdown): python tools/symbolic_repeat.py merged 4"""
import gc
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen

alg = sys.argv[1] if len(sys.argv) > 1 else "merged"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = pk.single_rank_context()
a, p = devgen.config_dist('cfg3', 1, 0, ctx.device)
torch.cuda.synchronize()
for algo in [alg] * reps:
    t = time.perf_counter()
    plan = pk.run_symbolic(a, p, algo, ctx)
    torch.cuda.synchronize()
    print(algo, 'symbolic wall ms', (time.perf_counter() - t) * 1e3, flush=True)
    del plan
    gc.collect()
    torch.cuda.synchronize()
