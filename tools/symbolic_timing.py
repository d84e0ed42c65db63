import sys, time, os
sys.path.insert(0, '/root/repo')
import torch
import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen
ctx = pk.single_rank_context()
a, p = devgen.config_dist('cfg3', 1, 0, ctx.device)
torch.cuda.synchronize()
for alg in ('allatonce', 'merged', 'allatonce'):
    t = time.perf_counter()
    plan = pk.run_symbolic(a, p, alg, ctx)
    torch.cuda.synchronize()
    print(alg, 'symbolic wall ms', (time.perf_counter() - t) * 1e3, flush=True)
    del plan
