"""Warm symbolic time of config 4 (block transport) at nn^3 nodes:
python tools/sym_cfg4.py [nn] [reps]"""
import gc
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems_amg as amg
from tools.bench_configs import upload

nn = int(sys.argv[1]) if len(sys.argv) > 1 else 96
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = pk.single_rank_context()
A, P = amg.block_transport(nn)
a, p = upload(A, P, ctx.device)
for _ in range(reps):
    gc.collect()
    torch.cuda.synchronize()
    t = time.perf_counter()
    plan = pk.run_symbolic(a, p, "allatonce", ctx)
    torch.cuda.synchronize()
    print("symbolic ms", (time.perf_counter() - t) * 1e3, flush=True)
    del plan
