"""Numeric passes of config 4 (block transport, smoothed aggregation; plan
maps) at a reduced node grid, for profiling: python tools/cfg4_numeric.py [nn] [reps]"""
import sys

sys.path.insert(0, '/root/repo')
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems_amg as amg
from tools.bench_configs import upload

nn = int(sys.argv[1]) if len(sys.argv) > 1 else 48
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = pk.single_rank_context()
A, P = amg.block_transport(nn)
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
