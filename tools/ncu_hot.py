"""Top SASS lines of an ncu report by stall samples, with the dominant stall
reasons: python tools/ncu_hot.py report.ncu-rep [n] [--kernel REGEX]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 25
ksel = ["-k", "regex:" + sys.argv[sys.argv.index("--kernel") + 1]] if "--kernel" in sys.argv else []
out = subprocess.run(["ncu", "-i", rep, *ksel, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r != hdr]
ix = {h: i for i, h in enumerate(hdr)}
samp = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[samp] or 0) for r in data)
agg = {s: sum(float(r[ix[s]] or 0) for r in data) for s in stalls}
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
data.sort(key=lambda r: -float(r[samp] or 0))
for r in data[:n]:
    top = sorted(((float(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{float(r[samp] or 0) / tot:6.1%} {r[ix['Address']]:>6} {r[ix['Source']][:60]:60s} " +
          " ".join(f"{s}:{v / tot:.1%}" for v, s in top if v))
