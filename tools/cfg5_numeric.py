"""Numeric passes of config 5 (kNN Laplacian, hash path by policy) at a
reduced point count, for profiling: python tools/cfg5_numeric.py [npts] [reps]"""
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems_amg as amg
from tools.bench_configs import upload

npts = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = pk.single_rank_context()
A, P = amg.knn_laplacian(npts)
a, p = upload(A, P, ctx.device)
plan = pk.run_symbolic(a, p, "allatonce", ctx)
torch.cuda.synchronize()
print("counters", plan.device_counters(), flush=True)
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pk.run_numeric_device(a, p, plan, ctx)
    e1.record()
    torch.cuda.synchronize()
    print("numeric ms", e0.elapsed_time(e1), flush=True)
