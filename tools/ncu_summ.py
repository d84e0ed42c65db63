"""Summarise an ncu report of a numeric kernel: per-row instruction and L1
wavefront budget, plus the top stall/wavefront SASS lines.
usage: python tools/ncu_summ.py report.ncu-rep [rows]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
nrows = float(sys.argv[2]) if len(sys.argv) > 2 else 256.0 ** 3


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
R = dict(zip(raw[0], raw[2]))
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_red.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
for k in want:
    v = R.get(k, "?")
    try:
        f = float(v.replace(",", ""))
        per = f / nrows
        print(f"{k:70s} {f:16.4g}   per-row {per:10.3f}")
    except ValueError:
        print(f"{k:70s} {v}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
hdr = src[1]; data = src[2:]
ix = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError):
        return 0.0


print("\ntop by stall samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:15]:
    print(f"  {r[ix['Source']][:58]:58} samp={f(r,'Warp Stall Sampling (All Samples)'):7.0f} inst/row={f(r,'Instructions Executed')/nrows:5.2f}")
print("\ntop by L1 wavefronts (shared) / tags (global)")
for r in sorted(data, key=lambda r: -(f(r, "L1 Wavefronts Shared") + f(r, "L1 Tag Requests Global")))[:15]:
    print(f"  {r[ix['Source']][:58]:58} inst/row={f(r,'Instructions Executed')/nrows:5.2f} shwf={f(r,'L1 Wavefronts Shared')/nrows:6.2f}"
          f" ideal={f(r,'L1 Wavefronts Shared Ideal')/nrows:5.2f} gtag={f(r,'L1 Tag Requests Global')/nrows:5.2f} l2s={f(r,'L2 Theoretical Sectors Global')/nrows:5.2f}")
