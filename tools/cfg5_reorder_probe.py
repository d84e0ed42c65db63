"""Upper bound of a plan-internal renumbering for config 5: time the hash
numeric pass on device-generated operands as given (natural point order) and
after renumbering the fine points in aggregate order (A symmetrically
permuted, P's rows permuted; C is unchanged).  python tools/cfg5_reorder_probe.py [npts]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen
from paper_1905_08423_b200.partition import DistMatrix, make_partition

npts = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
ctx = pk.single_rank_context()
dev = ctx.device
(arp, acol, aval), (prp, pcol, pval), nagg = devgen.gen_knn_laplacian(npts, dev)


def dist(arp, acol, aval, prp, pcol, pval):
    rp_a, rp_p = make_partition(npts, 1), make_partition(nagg, 1)
    a = DistMatrix(rp_a, rp_a, 0, devgen.split_rows_device(arp, acol, aval, 0, npts, 0, npts, npts))
    p = DistMatrix(rp_a, rp_p, 0, devgen.split_rows_device(prp, pcol, pval, 0, npts, 0, nagg, nagg))
    return a, p


def run(a, p, tag):
    for alg in ("allatonce", "two-step"):
        plan = pk.run_symbolic(a, p, alg, ctx)
        ms = []
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rp, col, v = pk.run_numeric_device(a, p, plan, ctx)
            e1.record()
            torch.cuda.synchronize()
            ms.append(round(e0.elapsed_time(e1), 2))
        print(tag, alg, "path", plan.device_counters()["numeric_path"], "numeric ms", ms, "sum", float(v.sum()), flush=True)
        del plan


run(*dist(arp, acol, aval, prp, pcol, pval), "natural  ")
# aggregate order: rows sorted by the first coarse column of P(i,:)
first = pcol[prp[:-1]].to(torch.int64)
order = torch.argsort(first * npts + torch.arange(npts, device=dev))
inv = torch.empty_like(order)
inv[order] = torch.arange(npts, device=dev)


def permute_rows(rp, col, val, order, colmap=None):
    ln = (rp[1:] - rp[:-1])[order]
    nrp = torch.zeros_like(rp)
    torch.cumsum(ln, 0, out=nrp[1:])
    src = torch.repeat_interleave(rp[:-1][order] - nrp[:-1], ln) + torch.arange(int(nrp[-1]), device=dev)
    ncol = col[src].to(torch.int64)
    nval = val[src]
    if colmap is not None:
        ncol = colmap[ncol]
        # sort columns inside rows
        rows = torch.repeat_interleave(torch.arange(npts, device=dev), ln)
        key = rows * npts + ncol
        o = torch.argsort(key)
        ncol, nval = ncol[o], nval[o]
    return nrp, ncol.to(torch.int32), nval


a2 = permute_rows(arp, acol, aval, order, inv)
p2 = permute_rows(prp, pcol, pval, order)
run(*dist(*a2, *p2), "aggregate")
