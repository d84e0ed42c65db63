"""Summarise an ncu report of a numeric kernel: per-row instruction and L1
wavefront budget, plus the top stall/wavefront SASS lines.
usage: python tools/ncu_summ.py report.ncu-rep [rows] [--kernel REGEX] [--write DESC OUT.txt]
(--kernel picks one kernel of a report that holds several)"""
import csv, io, os, subprocess, sys

rep = sys.argv[1]
nrows = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 256.0 ** 3
KSEL = ["-k", "regex:" + sys.argv[sys.argv.index("--kernel") + 1]] if "--kernel" in sys.argv else []


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *KSEL, *a], capture_output=True, text=True).stdout


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
hdr = src[1]; data = [r for r in src[2:] if len(r) == len(hdr) and r != hdr]
ix = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0


print("\ntop by stall samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:15]:
    print(f"  {r[ix['Source']][:58]:58} samp={f(r,'Warp Stall Sampling (All Samples)'):7.0f} inst/row={f(r,'Instructions Executed')/nrows:5.2f}")
print("\ntop by L1 wavefronts (shared) / tags (global)")
for r in sorted(data, key=lambda r: -(f(r, "L1 Wavefronts Shared") + f(r, "L1 Tag Requests Global")))[:15]:
    print(f"  {r[ix['Source']][:58]:58} inst/row={f(r,'Instructions Executed')/nrows:5.2f} shwf={f(r,'L1 Wavefronts Shared')/nrows:6.2f}"
          f" ideal={f(r,'L1 Wavefronts Shared Ideal')/nrows:5.2f} gtag={f(r,'L1 Tag Requests Global')/nrows:5.2f} l2s={f(r,'L2 Theoretical Sectors Global')/nrows:5.2f}")


def write_summary(rep_path, kernel_desc, out_json, out_txt, nrows_):
    """profiles/ncu_numeric_summary.json (read by bench.py for roofline.traffic)
    and a text summary of the same capture."""
    import json as _json
    raw_ = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep_path, *KSEL, "--page", "raw", "--csv"],
                                                      capture_output=True, text=True).stdout)))
    R_ = dict(zip(raw_[0], raw_[2]))
    U_ = dict(zip(raw_[0], raw_[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def g(k):
        try:
            return float(R_[k].replace(",", ""))
        except (KeyError, ValueError):
            return None

    def gb(k):  # bytes, whatever unit ncu chose for the column
        v = g(k)
        return None if v is None else v * scale.get(U_.get(k, "byte"), 1.0)
    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    unit_scale = 1.0
    d = {"kernel": kernel_desc,
         "capture": f"ncu --set full --clock-control none, 1 launch ({os.path.basename(out_txt)})",
         "gpu_time_ms": g("gpu__time_duration.sum"),
         "dram_bytes_read": rd * unit_scale if rd is not None else None,
         "dram_bytes_write": wr * unit_scale if wr is not None else None,
         "dram_bytes_per_launch": (rd + wr) * unit_scale if rd is not None and wr is not None else None,
         "l2_hit_rate_pct": g("lts__t_sector_hit_rate.pct"),
         "l1_data_pipe_lsu_wavefronts_pct": g("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
         "instructions": g("smsp__inst_executed.sum"),
         "rows": nrows_}
    with open(out_json, "w") as f:
        _json.dump(d, f, indent=1)
    return d


if __name__ == "__main__" and "--write" in sys.argv:
    import os
    w = sys.argv.index("--write")
    write_summary(rep, sys.argv[w + 1], "profiles/ncu_numeric_summary.json", sys.argv[w + 2], nrows)
