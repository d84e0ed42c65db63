"""Small all-at-once products for compute-sanitizer (memcheck / racecheck):
config 3 at 16^3 and 24^3 and config 1 at 16^3 through the class-lockstep
pass, the per-row pass, the deterministic pass and the single-shot pass.
compute-sanitizer --tool racecheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen

ctx = pk.single_rank_context()
for cfg, n in (("cfg3", 16), ("cfg3", 24), ("cfg1", 16)):
    a, p = devgen.config_dist(cfg, 1, 0, ctx.device, n_fine=n)
    ref = None
    for kw in ({}, {"lockstep": False}, {"deterministic": True}, {"single_shot": True}):
        plan = pk.run_symbolic(a, p, "allatonce", ctx, **kw)
        if not plan.values_ready:
            pk.run_numeric_device(a, p, plan, ctx)
        plan.check()
        rp, col, v = plan.c_device()
        torch.cuda.synchronize()
        if ref is None:
            ref = v.clone()
        print(cfg, n, kw, plan.device_counters()["numeric_path"], float((v - ref).abs().max()), flush=True)
        del plan
print("done")
