#!/usr/bin/env python
"""Benchmark of the B200 triple product on BASELINE.json config 3, level 1.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one numeric C = P^T A P pass (plan reused: the paper's 1 symbolic +
11 numeric protocol) on the 27-point random 256^3 operator with
trilinear P to 128^3 (config 3 level 1; z-slab row blocks over N GPUs,
torchrun one process per GPU over NCCL).  Inputs are generated on the device
and are larger than L2 (A alone is 5.5 GB), so no flush is needed between
steps.  The line reports:

  value      GFLOP/s of the all-at-once numeric pass, 2 flops per multiply-add
             of the triple product (MAC_AP + MAC_outer), whole job
  e2e        the same metric through the public API (run_numeric) with host
             buffers: H2D of the step's A/P values, D2H of C's values
  roofline   HBM: algorithmic bytes (A + P + C in the device layout) per launch
             of the fused numeric kernel / its CUDA-event time vs MEASURED_PEAKS
  variants   merged and two-step numeric times, symbolic times, aux memory
  cpu_baseline  the CPU oracle port (oracle/) on a bounded sample, rank 0, N=1

``--impl reference`` times the reference algorithm on the host cores instead
(the C port of the reference in oracle/, one simulated rank per thread; the
reference itself is Python and cannot travel to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PtAP GFLOP/s & achieved HBM GB/s at 1/2/4/8 B200; peak auxiliary memory"
UNIT = "GFLOP/s"
SAMPLE_PLANES = 32  # CPU sample: fine z-planes [0, 32) of config 3 level 1


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--n-fine", type=int, default=None, help="override grid size (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--csv", default=None, help="also write the reference bench's CSV columns (src/bench.py:43-56) "
                                                  "plus GFLOP/s, GB/s and roofline, one row per algorithm")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML sampling thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index=0, period=0.01):
        self.samples, self.reasons = [], set()
        self.period, self.index = period, index
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of the fused numeric kernel from the committed
    ncu --set full summary, when one exists."""
    path = os.path.join(ROOT, "profiles", "ncu_numeric_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


# ---------------------------------------------------------------------------
# CPU legs (oracle port) -- test/bench infrastructure only
# ---------------------------------------------------------------------------
def cpu_sample_operands(planes=SAMPLE_PLANES, n=256, seed=None):
    """Host CSR of the fine rows of z-planes [0, planes) of config 3 level 1:
    A rows [0, R) (columns up to the next plane) padded to R + n^2 rows and
    P rows [0, R + n^2), so P^T A P equals the contribution of those rows."""
    import numpy as np

    from paper_1905_08423_b200 import problems as gen
    from paper_1905_08423_b200.sparse import CsrMatrix

    spec = gen.CONFIGS["cfg3"]
    R = planes * n * n
    ns = R + n * n
    a = gen.random27(n, spec.seed if seed is None else seed, 0, R)
    a_ip = np.concatenate((a.row_offsets, np.full(ns - R, a.row_offsets[-1])))
    A = CsrMatrix(ns, ns, a_ip, a.col_indices, a.values, check=False)
    p = gen.trilinear(n // 2, 0, ns)
    return A, p


def run_cpu_oracle(nthreads=1, steps=1, planes=SAMPLE_PLANES):
    from oracle import oracle as orc

    os.environ["OMP_NUM_THREADS"] = str(nthreads)
    A, P = cpu_sample_operands(planes)
    plan = orc.OraclePlan(A.nrows, P.ncols, A.row_offsets, A.col_indices, P.row_offsets, P.col_indices,
                          nranks=nthreads, algorithm="allatonce")
    times = []
    out = None
    for _ in range(steps):
        t0 = time.perf_counter()
        out = plan.numeric(A.values, P.values, out)
        times.append(time.perf_counter() - t0)
    st = plan.num_stats
    mac = int(st.mac_ap + st.mac_outer)
    return {"times": times, "mac": mac, "rows": int(planes * 256 * 256), "nnz_c": plan.nnz}


def reference_arm(args):
    """--impl reference: the reference algorithm (C port) on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc

    orc.build()
    threads = os.cpu_count() or 1
    total = args.steps + args.warmup
    res = run_cpu_oracle(nthreads=threads, steps=total)
    times = res["times"][args.warmup:] or res["times"]
    t = statistics.median(times)
    value = 2.0 * res["mac"] / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg3 L1 sample: fine z-planes [0,{SAMPLE_PLANES}) of 256^3 27-pt random, trilinear P, "
                               "numeric all-at-once", "sample_rows": res["rows"], "mac": res["mac"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"fine z-planes [0,{SAMPLE_PLANES}) of config 3 level 1 ({res['rows']} rows), "
                                   f"one simulated reference rank per thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def alg_bytes(a, p, c_nnz, ncl):
    """Algorithmic HBM bytes of one numeric pass in the device layout:
    A and P read once (int64 row offsets, int32 columns, fp64 values), C's
    structure read and values written once."""
    def csr_bytes(d):
        return d.row_ptr.numel() * 8 + d.nnz * 12

    return (csr_bytes(a.local.diag) + csr_bytes(a.local.offdiag) + csr_bytes(p.local.diag)
            + csr_bytes(p.local.offdiag) + (ncl + 1) * 8 + c_nnz * 12)


def time_numeric(pk, a, p, plan, ctx, steps, warmup, torch, kernel_events=None):
    """Per-step device time of numeric passes (events on the launching stream)."""
    import ctypes

    from paper_1905_08423_b200 import _lib

    L = _lib.load()
    st = plan._ops.struct()
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)

    def one():
        if ctx.nranks > 1:
            pk.run_numeric_device(a, p, plan, ctx)
            return None
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        _lib.check(L.ptap_numeric_send(plan._h, ctypes.byref(st), sp))
        e0.record(stream)
        _lib.check(L.ptap_numeric_local(plan._h, ctypes.byref(st), sp))
        e1.record(stream)
        return (e0, e1)

    for _ in range(warmup):
        one()
    _lib.check(L.ptap_plan_check(plan._h, sp))
    ctx.barrier()
    torch.cuda.synchronize()
    launches0 = plan.device_counters()["kernel_launches"]
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    evs = [one() for _ in range(steps)]
    stop.record(stream)
    torch.cuda.synchronize()
    ctx.barrier()
    _lib.check(L.ptap_plan_check(plan._h, sp))
    launches = plan.device_counters()["kernel_launches"] - launches0
    total_ms = start.elapsed_time(stop)
    kern = [e0.elapsed_time(e1) for (e0, e1) in evs if e0 is not None] if evs and evs[0] is not None else []
    return total_ms / steps, kern, launches


def row_scaled_diff(rp_a, val_a, rp_b, val_b, torch):
    """max over entries of |a - b| / max_k |a_ik| (SURVEY §8(c) values B);
    inf if the two patterns' row offsets differ."""
    if rp_a.numel() != rp_b.numel() or not torch.equal(rp_a, rp_b):
        return float("inf")
    n = rp_a.numel() - 1
    if val_a.numel() == 0:
        return 0.0
    rows = torch.repeat_interleave(torch.arange(n, device=rp_a.device), rp_a[1:] - rp_a[:-1])
    scale = torch.zeros(n, dtype=torch.float64, device=rp_a.device)
    scale.scatter_reduce_(0, rows, val_a.abs(), reduce="amax")
    d = (val_a - val_b).abs() / scale[rows].clamp_min(1e-300)
    return float(d.max().item())


def write_csv(path, line, out, ctx):
    """The reference bench's CSV columns (src/bench.py:43-56) plus this
    bench's rates, one row per algorithm."""
    import csv
    cols = ["np", "algorithm", "mem_input", "mem_output", "mem_aux", "mem_transient_peak", "mem_plan",
            "time_sym_s", "time_num_s", "time_total_s", "repeats", "verified",
            "gflops", "alg_gbs", "roofline_frac", "n_gpus"]
    mac2 = 2.0 * line["config"]["mac_total"]
    alg_bytes = line["roofline"]["alg_bytes_per_launch"] * ctx.nranks
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(cols)
        for alg, v in out.items():
            mem = v["memory"]["peak"]
            t_num = v["numeric_ms"] * 1e-3
            diff = v.get("row_scaled_diff_vs_allatonce", 0.0)
            w.writerow([ctx.nranks, alg, mem["input_matrices"], mem["output_matrix"], mem["auxiliary_matrices"],
                        mem["transient_hash_peak"], mem["plan_cache"], v["symbolic_ms"] * 1e-3, t_num,
                        v["symbolic_ms"] * 1e-3 + t_num, line["steps"], bool(diff <= 1e-12),
                        mac2 / t_num / 1e9, alg_bytes / t_num / 1e9,
                        alg_bytes / t_num / 1e9 / (line["roofline"]["peak"] * ctx.nranks), ctx.nranks])


def max_over_ranks(x, ctx, torch):
    if ctx.nranks == 1:
        return x
    t = torch.tensor([float(x)], dtype=torch.float64, device=ctx.device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, ctx, torch):
    if ctx.nranks == 1:
        return x
    t = torch.tensor([float(x)], dtype=torch.float64, device=ctx.device)
    torch.distributed.all_reduce(t)
    return float(t.item())


def our_arm(args):
    import numpy as np
    import torch

    import paper_1905_08423_b200 as pk
    from paper_1905_08423_b200 import devgen

    ctx = pk.init_from_env()
    dev = ctx.device
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a, p = devgen.config_dist(args.config, ctx.nranks, ctx.rank, dev, n_fine=args.n_fine)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    out = {}

    def symbolic(alg):
        torch.cuda.synchronize()
        ctx.barrier()
        t = time.perf_counter()
        plan = pk.run_symbolic(a, p, alg, ctx)
        torch.cuda.synchronize()
        ctx.barrier()
        return plan, max_over_ranks(time.perf_counter() - t, ctx, torch)

    # --- headline: all-at-once ------------------------------------------------
    import gc

    def warm_symbolic(alg):
        """cold call (one-time module and memory-pool setup), then three warm
        calls; the warm figure is the fastest (the host-side driver calls
        occasionally stall for tens of ms on these boxes; all are reported)"""
        pl, cold = symbolic(alg)
        warm = []
        for _ in range(3):
            del pl
            gc.collect()
            torch.cuda.synchronize()
            pl, t = symbolic(alg)
            warm.append(t)
        return pl, cold, min(warm), warm

    plan, sym_cold, sym_s, sym_all = warm_symbolic("allatonce")
    cnt = plan.device_counters()
    mac = sum_over_ranks(cnt["mac_ap"] + cnt["mac_outer"], ctx, torch)
    flops = 2.0 * mac
    c_rp, c_col, c_val = plan.c_device()
    ncl = c_rp.numel() - 1
    my_bytes = alg_bytes(a, p, c_col.numel(), ncl)
    clocks = ClockSampler(index=dev.index or 0)
    with clocks:
        ms, kern_ms, launches = time_numeric(pk, a, p, plan, ctx, args.steps, args.warmup, torch)
    ms = max_over_ranks(ms, ctx, torch)
    value = flops / (ms * 1e-3) / 1e9
    mem = plan.memory()
    peak, peak_src = measured_peak_hbm()
    traffic, ncu_meta = ncu_traffic()
    kms = statistics.mean(kern_ms) if kern_ms else ms
    achieved = my_bytes / (kms * 1e-3) / 1e9
    out["allatonce"] = {"numeric_ms": ms, "symbolic_ms": sym_s * 1e3, "symbolic_cold_ms": sym_cold * 1e3,
                        "symbolic_warm_runs_ms": [t * 1e3 for t in sym_all],
                        "ptap_wall_ms": sym_s * 1e3 + ms,
                        "aux_peak_bytes": mem["device_high_water"] - mem["current"]["output_matrix"],
                        "memory": mem}

    # --- config 3 level 2: A2 = C1 kept on the device (hierarchy driver), P2 trilinear
    level2 = None
    if args.config == "cfg3" and not args.no_variants:
        try:
            from paper_1905_08423_b200.hierarchy import _coarse_operator
            from paper_1905_08423_b200.partition import DistMatrix, make_partition
            n2 = (args.n_fine or 256) // 2
            m2 = (n2 // 2) ** 3
            cp2 = make_partition(m2, ctx.nranks)
            a2, _, _ = _coarse_operator(plan, p)
            lo2, hi2 = a2.row_part.owned_range(ctx.rank)
            clo2, chi2 = cp2.owned_range(ctx.rank)
            prp, pcol, pval = devgen.gen_trilinear_rows(n2 // 2, lo2, hi2, dev)
            p2 = DistMatrix(a2.row_part, cp2, ctx.rank,
                            devgen.split_rows_device(prp, pcol, pval, lo2, hi2, clo2, chi2, m2))
            t = time.perf_counter()
            plan2 = pk.run_symbolic(a2, p2, "allatonce", ctx)
            torch.cuda.synchronize()
            s2 = time.perf_counter() - t
            ms2, _, _ = time_numeric(pk, a2, p2, plan2, ctx, max(3, args.steps // 2), 2, torch)
            c2 = plan2.device_counters()
            level2 = {"numeric_ms": max_over_ranks(ms2, ctx, torch), "symbolic_ms": s2 * 1e3, "nnz_c": c2["nnz_c"],
                      "gflops": 2.0 * (c2["mac_ap"] + c2["mac_outer"]) / (ms2 * 1e-3) / 1e9,
                      "driver": "paper_1905_08423_b200.hierarchy (A2 = C1 on the device)"}
            del plan2
        except Exception as exc:  # report, do not fail the headline line
            level2 = {"error": repr(exc)}

    # --- e2e through the public API with host buffers ---------------------------
    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(pk, a, p, plan, ctx, flops, max(3, min(args.steps, 5)), torch)

    # --- variants (headline plan released first so every variant's warm
    # symbolic phase sees the same memory pool state) -----------------------------
    # the all-at-once C is kept to cross-check the variants on the device
    c_rp_ref, c_val_ref = (c_rp.clone(), c_val.clone()) if not args.no_variants else (None, None)
    del plan, c_rp, c_col, c_val
    gc.collect()
    torch.cuda.synchronize()
    if not args.no_variants:
        for alg in ("merged", "two-step"):
            vplan, vcold, vsym, vall = warm_symbolic(alg)
            vms, _, _ = time_numeric(pk, a, p, vplan, ctx, max(3, args.steps // 2), 2, torch)
            vmem = vplan.memory()
            vms = max_over_ranks(vms, ctx, torch)
            vrp, _, vval = vplan.c_device()
            diff = max_over_ranks(row_scaled_diff(c_rp_ref, c_val_ref, vrp, vval, torch), ctx, torch)
            out[alg] = {"numeric_ms": vms, "symbolic_ms": vsym * 1e3, "symbolic_cold_ms": vcold * 1e3,
                        "symbolic_warm_runs_ms": [t * 1e3 for t in vall],
                        "ptap_wall_ms": vsym * 1e3 + vms,
                        "aux_peak_bytes": vmem["device_high_water"] - vmem["current"]["output_matrix"],
                        "row_scaled_diff_vs_allatonce": diff,
                        "memory": vmem}
            del vplan, vrp, vval
            gc.collect()
            torch.cuda.synchronize()
        del c_rp_ref, c_val_ref

    # --- CPU baseline (rank 0, N = 1) -----------------------------------------
    cpu = None
    if ctx.rank == 0 and ctx.nranks == 1 and not args.no_cpu_baseline:
        res = run_cpu_oracle(nthreads=1, steps=1)
        t = res["times"][0]
        cpu = {"value": 2.0 * res["mac"] / t / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"fine z-planes [0,{SAMPLE_PLANES}) of config 3 level 1 ({res['rows']} rows, "
                         f"{res['mac']} MAC), oracle all-at-once numeric pass, np=1, 1 thread",
               "seconds": t, "host_cores_available": os.cpu_count()}

    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ctx.nranks, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} L1: 27-pt random {args.n_fine or 256}^3 -> trilinear "
                                   f"{(args.n_fine or 256) // 2}^3, numeric all-at-once (plan reused)",
                       "parallelism": f"z-slab row blocks x{ctx.nranks}", "mac_total": int(mac),
                       "flops_per_mac": 2, "l2": "inputs larger than L2 (A = %.1f GB), no flush" % (my_bytes / 1e9),
                       "gen_s": gen_s},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "k_outer_numeric_q4a (ptap_numeric_local)", "kernel_ms": kms,
                         "alg_bytes_per_launch": my_bytes},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "variants": {k: {kk: vv for kk, vv in v.items() if kk != "memory"} for k, v in out.items()},
            "memory_bytes": {k: v["memory"] for k, v in out.items()},
            "level2": level2,
        }
        if "two-step" in out:
            line["variants"]["allatonce_over_two_step_time"] = out["allatonce"]["numeric_ms"] / out["two-step"]["numeric_ms"]
        print(json.dumps(line))
        if args.csv:
            write_csv(args.csv, line, out, ctx)
    if ctx.nranks > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def e2e_leg(pk, a, p, plan, ctx, flops, steps, torch):
    """run_numeric through the public API with host DistMatrix operands whose
    values live in pinned host memory: every step uploads A's and P's values,
    runs the pass and downloads C's values."""
    import numpy as np

    from paper_1905_08423_b200.partition import DistMatrix, LocalMatrix
    from paper_1905_08423_b200.sparse import CsrMatrix

    def host_local(dl):
        def blk(d):
            vals = torch.empty(d.nnz, dtype=torch.float64, pin_memory=True)
            vals.copy_(d.val)
            return CsrMatrix(d.nrows, d.ncols, d.row_ptr.cpu().numpy(), d.col.cpu().numpy(), vals.numpy(), check=False)
        return LocalMatrix(dl.row_lo, dl.row_hi, dl.col_lo, dl.col_hi, blk(dl.diag), blk(dl.offdiag),
                           dl.col_map.cpu().numpy().astype(np.int64))

    ah = DistMatrix(a.row_part, a.col_part, a.rank, host_local(a.local))
    ph = DistMatrix(p.row_part, p.col_part, p.rank, host_local(p.local))
    # the plan's device operands become the upload targets
    from paper_1905_08423_b200.tripleproduct import _identity
    from paper_1905_08423_b200.device import structure_token
    plan._a_token = (_identity(ah.local), None)
    plan._p_token = (_identity(ph.local), None)
    h2d = (ah.local.diag.nnz + ah.local.offdiag.nnz + ph.local.diag.nnz + ph.local.offdiag.nnz) * 8
    pk.run_numeric(ah, ph, plan, ctx)  # warm
    torch.cuda.synchronize()
    ctx.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        c = pk.run_numeric(ah, ph, plan, ctx)
    torch.cuda.synchronize()
    ctx.barrier()
    dt = max_over_ranks((time.perf_counter() - t0) / steps, ctx, torch)
    d2h = (c.diag.nnz + c.offdiag.nnz) * 8
    # restore device operands for anything that follows
    plan._a_dev, plan._p_dev = a.local, p.local
    plan._ops.a, plan._ops.p = a.local, p.local
    return {"value": flops / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": dt * 1e3, "api": "paper_1905_08423_b200.run_numeric(host DistMatrix, pinned values)"}


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
