"""cProfile of the host side of run_symbolic (device operands, cfg3 L1)."""
import cProfile
import gc
import pstats
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen

ALG = sys.argv[1] if len(sys.argv) > 1 else "allatonce"
ctx = pk.single_rank_context()
a, p = devgen.config_dist('cfg3', 1, 0, ctx.device)
torch.cuda.synchronize()
for _ in range(2):
    plan = pk.run_symbolic(a, p, ALG, ctx)
    del plan
    gc.collect()
torch.cuda.synchronize()
pr = cProfile.Profile()
for _ in range(3):
    t = time.perf_counter()
    pr.enable()
    plan = pk.run_symbolic(a, p, ALG, ctx)
    torch.cuda.synchronize()
    pr.disable()
    print("wall ms", (time.perf_counter() - t) * 1e3)
    del plan
    gc.collect()
    torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
