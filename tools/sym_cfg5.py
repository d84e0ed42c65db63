"""Warm symbolic time of config 5 (kNN Laplacian) at npts points: python tools/sym_cfg5.py npts"""
import sys, time, gc
sys.path.insert(0, '/root/repo')
import torch
import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems_amg as amg
from tools.bench_configs import upload
ctx = pk.single_rank_context()
A, P = amg.knn_laplacian(int(sys.argv[1]))
a, p = upload(A, P, ctx.device)
for r in range(3):
    gc.collect(); torch.cuda.synchronize()
    t = time.perf_counter()
    plan = pk.run_symbolic(a, p, "allatonce", ctx)
    torch.cuda.synchronize()
    print("symbolic ms", (time.perf_counter() - t) * 1e3, flush=True)
    del plan
