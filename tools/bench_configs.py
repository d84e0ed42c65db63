"""Every BASELINE.json config at its full size on one B200: numeric and
symbolic time, GFLOP/s, algorithmic GB/s and roofline fraction, peak
auxiliary device memory, for all-at-once, merged and two-step; merged and
two-step C cross-checked against all-at-once on the device, and all-at-once C
checked against the CPU oracle (pattern exact, row-scaled values <= 1e-12)
where --oracle names the config.

usage: python tools/bench_configs.py [--configs cfg1,cfg2,cfg3,cfg3l2,cfg4,cfg5]
                                     [--oracle cfg1,cfg2,cfg4,cfg5] [--reps 11]
                                     [--cfg4-nn 96] [--cfg5-npts 20000000]
One JSON line per config on stdout.  The oracle (oracle/) is the checker
here, never the measured path.
"""
import argparse
import gc
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen
from paper_1905_08423_b200 import problems as gen
from paper_1905_08423_b200.partition import DistMatrix, make_partition

ALGS = ("allatonce", "merged", "two-step")


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def upload(A, P, dev):
    """Host CsrMatrix pair -> single-rank device DistMatrix pair."""
    def up(M):
        rp = torch.as_tensor(np.ascontiguousarray(M.row_offsets, np.int64), device=dev)
        col = torch.as_tensor(np.ascontiguousarray(M.col_indices, np.int32), device=dev)
        val = torch.as_tensor(np.ascontiguousarray(M.values, np.float64), device=dev)
        return devgen.split_rows_device(rp, col, val, 0, M.nrows, 0, M.ncols, M.ncols)

    rp_a, rp_p = make_partition(A.nrows, 1), make_partition(P.ncols, 1)
    return DistMatrix(rp_a, rp_a, 0, up(A)), DistMatrix(rp_a, rp_p, 0, up(P))


def host_copy(a, p):
    """Host CsrMatrix copies of single-rank device operands (oracle input)."""
    from paper_1905_08423_b200.sparse import CsrMatrix

    def down(d):
        return CsrMatrix(d.nrows, d.ncols, d.row_ptr.cpu().numpy(), d.col.cpu().numpy().astype(np.int64),
                         d.val.cpu().numpy(), check=False)

    return down(a.local.diag), down(p.local.diag)


def csr_bytes(d):
    return d.row_ptr.numel() * 8 + d.nnz * 12


def row_scaled(rp, ref, got):
    n = rp.numel() - 1
    if ref.numel() == 0:
        return 0.0
    rows = torch.repeat_interleave(torch.arange(n, device=rp.device), rp[1:] - rp[:-1])
    scale = torch.zeros(n, dtype=torch.float64, device=rp.device)
    scale.scatter_reduce_(0, rows, ref.abs(), reduce="amax")
    return float(((ref - got).abs() / scale[rows].clamp_min(1e-300)).max().item())


def measure(a, p, reps, ctx):
    out = {}
    ref = None
    peak = peak_hbm()
    in_bytes = csr_bytes(a.local.diag) + csr_bytes(a.local.offdiag) + csr_bytes(p.local.diag) + csr_bytes(p.local.offdiag)
    for alg in ALGS:
        gc.collect()
        torch.cuda.synchronize()
        t = time.perf_counter()
        plan = pk.run_symbolic(a, p, alg, ctx)
        torch.cuda.synchronize()
        cold = time.perf_counter() - t
        del plan
        gc.collect()
        torch.cuda.synchronize()
        t = time.perf_counter()
        plan = pk.run_symbolic(a, p, alg, ctx)
        torch.cuda.synchronize()
        sym = time.perf_counter() - t
        pk.run_numeric_device(a, p, plan, ctx)
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pk.run_numeric_device(a, p, plan, ctx)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        cnt = plan.device_counters()
        mac = cnt["mac_ap"] + cnt["mac_outer"]
        mem = plan.memory()
        c_rp, c_col, c_val = plan.c_device()
        alg_b = in_bytes + c_rp.numel() * 8 + c_col.numel() * 12
        r = {"numeric_ms": ms, "symbolic_ms": sym * 1e3, "symbolic_cold_ms": cold * 1e3,
             "ptap_wall_ms": sym * 1e3 + ms, "gflops": 2.0 * mac / (ms * 1e-3) / 1e9,
             "alg_gbs": alg_b / (ms * 1e-3) / 1e9, "roofline_frac": alg_b / (ms * 1e-3) / 1e9 / peak,
             "aux_peak_bytes": mem["device_high_water"] - mem["current"]["output_matrix"],
             "plan_cache_bytes": mem["current"]["plan_cache"], "mac": mac, "nnz_c": int(c_col.numel()),
             "numeric_path": ("plan maps" if cnt["numeric_path"] else "hash") if alg != "two-step" else "two-step",
             "map_bytes": cnt["map_bytes"], "row_structures_ppm": cnt["row_structures_ppm"]}
        if ref is None:
            ref = (c_rp.clone(), c_col.clone(), c_val.clone())
        else:
            same = torch.equal(ref[0], c_rp) and torch.equal(ref[1], c_col)
            r["pattern_equal_allatonce"] = bool(same)
            r["row_scaled_diff_vs_allatonce"] = row_scaled(ref[0], ref[2], c_val) if same else float("inf")
        out[alg] = r
        del plan, c_rp, c_col, c_val
    out["allatonce_over_two_step_time"] = out["allatonce"]["numeric_ms"] / out["two-step"]["numeric_ms"]
    out["allatonce_over_two_step_aux"] = out["allatonce"]["aux_peak_bytes"] / max(out["two-step"]["aux_peak_bytes"], 1)
    return out, ref


def oracle_check(A, P, ref):
    from oracle.oracle import OraclePlan

    t = time.perf_counter()
    plan = OraclePlan(A.nrows, P.ncols, A.row_offsets, A.col_indices, P.row_offsets, P.col_indices,
                      nranks=1, algorithm="allatonce")
    val = plan.numeric(A.values, P.values)
    dt = time.perf_counter() - t
    rp, col, v = (x.cpu().numpy() for x in ref)
    pat = np.array_equal(rp, plan.row_ptr) and np.array_equal(col, plan.col)
    err = float("inf")
    if pat and val.size:
        rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
        scale = np.zeros(rp.size - 1)
        np.maximum.at(scale, rows, np.abs(val))
        err = float((np.abs(v - val) / np.maximum(scale[rows], 1e-300)).max())
    elif pat:
        err = 0.0
    return {"pattern_exact": bool(pat), "row_scaled_err": err, "oracle_s": dt, "ok": bool(pat and err <= 1e-12)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg3l2,cfg4,cfg5")
    ap.add_argument("--oracle", default="cfg1,cfg2,cfg4,cfg5")
    ap.add_argument("--reps", type=int, default=11)
    ap.add_argument("--cfg4-nn", type=int, default=96)
    ap.add_argument("--cfg5-npts", type=int, default=20_000_000)
    args = ap.parse_args()
    ctx = pk.single_rank_context()
    dev = ctx.device
    want_oracle = set(args.oracle.split(",")) if args.oracle else set()
    for name in args.configs.split(","):
        t = time.perf_counter()
        host = None
        if name in ("cfg1", "cfg2", "cfg3"):
            a, p = devgen.config_dist(name, 1, 0, dev)
            desc = gen.CONFIGS[name].name + (" level 1" if name == "cfg3" else "")
            if name in want_oracle:
                host = gen.config_operands(gen.CONFIGS[name])
        elif name == "cfg3l2":
            # level 2: A2 = C1 of level 1 (device), P2 trilinear 128^3 -> 64^3
            a1, p1 = devgen.config_dist("cfg3", 1, 0, dev)
            plan1 = pk.run_symbolic(a1, p1, "allatonce", ctx)
            pk.run_numeric_device(a1, p1, plan1, ctx)
            c_rp, c_col, c_val = plan1.c_device()
            m1 = 128 ** 3
            a = DistMatrix(make_partition(m1, 1), make_partition(m1, 1), 0,
                           devgen.split_rows_device(c_rp.clone(), c_col.clone(), c_val.clone(), 0, m1, 0, m1, m1))
            del plan1, a1, p1, c_rp, c_col, c_val
            prp, pcol, pval = devgen.gen_trilinear_rows(64, 0, m1, dev)
            p = DistMatrix(make_partition(m1, 1), make_partition(64 ** 3, 1), 0,
                           devgen.split_rows_device(prp, pcol, pval, 0, m1, 0, 64 ** 3, 64 ** 3))
            desc = "cfg3 level 2: A2 = C1 (128^3, 27-pt Galerkin), trilinear to 64^3"
        elif name == "cfg4":
            # generated on the device (csrc/ptap_gen.cu); the oracle gets a host copy
            a, p = devgen.block_transport_dist(args.cfg4_nn, 1, 0, dev)
            desc = f"cfg4: block transport {args.cfg4_nn}^3 nodes x 10, smoothed aggregation (device-generated)"
            if name in want_oracle:
                host = host_copy(a, p)
        elif name == "cfg5":
            a, p = devgen.knn_laplacian_dist(args.cfg5_npts, 1, 0, dev)
            torch.cuda.empty_cache()
            desc = f"cfg5: 26-NN Laplacian, {args.cfg5_npts} points, greedy aggregation (device-generated)"
            if name in want_oracle:
                host = host_copy(a, p)
        else:
            raise SystemExit(f"unknown config {name}")
        gen_s = time.perf_counter() - t
        line = {"config": name, "workload": desc, "n": a.local.diag.nrows, "m": p.col_part.nglobal,
                "nnz_a": a.local.diag.nnz + a.local.offdiag.nnz, "nnz_p": p.local.diag.nnz + p.local.offdiag.nnz,
                "gen_s": gen_s, "flops_per_mac": 2, "device": torch.cuda.get_device_name(0)}
        res, ref = measure(a, p, args.reps, ctx)
        line.update(res)
        if name in want_oracle and host is not None:
            line["oracle_allatonce_np1"] = oracle_check(host[0], host[1], ref)
        del a, p, ref, host
        gc.collect()
        torch.cuda.empty_cache()
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
