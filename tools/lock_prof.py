"""Profiling driver: config 3 level 1 (default 256^3), one symbolic phase and a
few all-at-once numeric passes on the default plan.  python tools/lock_prof.py [n] [passes]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = pk.single_rank_context()
a, p = devgen.config_dist("cfg3", 1, 0, ctx.device, n_fine=n)
plan = pk.run_symbolic(a, p, "allatonce", ctx)
ms = []
for r in range(passes):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pk.run_numeric_device(a, p, plan, ctx)
    e1.record()
    torch.cuda.synchronize()
    ms.append(round(e0.elapsed_time(e1), 3))
print("path", plan.device_counters()["numeric_path"], "numeric ms", ms, flush=True)
